"""GPU parity: libosam.so (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE north_star): relative L2 <= 1e-10 per subdomain and field after
the last step, and identical per-step Schwarz iteration counts.
"""
import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, opinf, schwarz

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(autouse=True)
def tiled_k1(monkeypatch):
    """These cases exercise the TMA-streamed tiled K1 at small sizes: force it (OSAM_GATHER_MAX=0); the
    small-subdomain gather path (K1S) has its own module, tests/test_gpu_small_path.py."""
    monkeypatch.setenv("OSAM_GATHER_MAX", "0")


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam, problem
    osam.lib()
    return problem


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def oracle_run(cfg, n_steps, rom_ops=None, e=None, every=None):
    models = schwarz.build_models(cfg, rom_ops=rom_ops, e_scale=e)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    snaps = {}

    def cb(k, st):
        if every and (k + 1) in every:
            snaps[k + 1] = [dict((kk, vv.copy()) for kk, vv in s.items()) for s in st]
    states, iters = schwarz.run(models, u0s, cfg["dt"], n_steps, cfg["tol"], cfg["max_iters"], cfg["min_iters"],
                                callback=cb)
    return models, states, iters, snaps


def compare(problem, subs, models, states, tol=TOL):
    worst = 0.0
    for sub, m, st in zip(subs, models, states):
        if m.kind == "fom":
            u, v, a = problem.fom_state(sub, accel=True)
            for got, ref in ((u, st["u"][0]), (v, st["v"][0]), (a, st["a"][0])):
                e = rel(got, ref)
                worst = max(worst, e)
                assert e <= tol, (m.spec["name"], e)
        else:
            uh, vh, ah = problem.rom_state(sub, accel=True)
            for got, ref in ((uh, st["uh"]), (vh, st["vh"]), (ah, st["ah"])):
                for b in range(ref.shape[0]):
                    e = rel(got[b], ref[b])
                    worst = max(worst, e)
                    assert e <= tol, (m.spec["name"], b, e)
    return worst


def run_both(problem, cfg, n_steps, rom_ops=None, checkpoints=()):
    e = problem.e_scale(cfg)
    subs = problem.build(cfg, rom_ops)
    problem.set_ics(cfg, subs, device="cuda:0")
    models, states, it_ref, snaps = oracle_run(cfg, n_steps, rom_ops, e, every=set(checkpoints))
    done = 0
    iters = []
    for cp in sorted(set(checkpoints) | {n_steps}):
        _, it = problem.run(cfg, subs, n_steps=cp - done)
        iters.append(it)
        done = cp
        if cp in snaps:
            compare(problem, subs, models, snaps[cp])
    iters = np.concatenate(iters)
    assert np.array_equal(iters, it_ref.reshape(iters.shape)), "Schwarz iteration counts differ"
    worst = compare(problem, subs, models, states)
    return subs, iters, worst


def test_c1_full_horizon(gpu):
    cfg = I.config("c1")
    _, iters, worst = run_both(gpu, cfg, cfg["n_steps"], checkpoints=(1, 10, 100))
    assert (iters == 3).all()
    print("c1 worst rel L2", worst)


@pytest.fixture(scope="module")
def c2_ops():
    return opinf.train(I.config("c2"), I)


def test_c2_fom_rom_full_horizon(gpu, c2_ops):
    cfg = I.config("c2")
    _, iters, worst = run_both(gpu, cfg, cfg["n_steps"], rom_ops=c2_ops, checkpoints=(1, 100))
    assert (iters == 3).all()
    print("c2 worst rel L2", worst)


def test_c5_batched_rom_rom(gpu):
    cfg = I.config("c5")
    ops = opinf.train(cfg, I)
    _, iters, worst = run_both(gpu, cfg, cfg["n_steps"], rom_ops=ops, checkpoints=(1, 200))
    assert iters.shape == (cfg["n_steps"], 64) and (iters == 3).all()
    print("c5 worst rel L2", worst)


@pytest.mark.parametrize("factor,steps", [(8.0, 25), (5.3, 12)])
def test_scaled_c3_several_tiles_ragged(gpu, factor, steps):
    """Non-matching meshes spanning several 32x8x16 interior tiles with ragged tails."""
    cfg = I.scaled(I.config("c3"), factor)
    _, iters, worst = run_both(gpu, cfg, steps, checkpoints=(1,))
    assert (iters == 3).all()


def test_scaled_c4_fom_between_two_roms(gpu):
    """Three subdomains: ROM | FOM | ROM, the FOM with two Schwarz faces (c4 topology)."""
    cfg = I.scaled(I.config("c4"), 10.0)
    cfg["rom"] = dict(cfg["rom"], r=40)
    cfg["rom"]["training"] = dict(cfg["rom"]["training"], n_steps=120,
                                  subdomains=[dict(s, kind="fom", nel=(8, 8, 8)) for s in cfg["subdomains"]])
    for s in cfg["subdomains"]:
        if s["kind"] == "rom":
            s["nel"] = (8, 8, 8)
    ops = opinf.train(cfg, I)
    run_both(gpu, cfg, 40, rom_ops=ops, checkpoints=(1,))


@pytest.mark.parametrize("nel", [(1, 1, 1), (3, 2, 5), (40, 9, 3)])
def test_single_fom_degenerate_and_ragged(gpu, nel):
    sub = I._sub("one", "fom", (0, 0, 0), (0.3, 0.2, 0.1), nel, (I.CLAMP, 0, 2, 0, 0, 4))
    cfg = dict(I.config("c1"), subdomains=[sub])
    cfg["ic"] = dict(kind="gauss3d", A=1e-3, sigma=0.05, center=(0.1, 0.1, 0.05), direction=(0.6, 0.0, 0.8))
    cfg["dt"] = 0.5 * min(0.3 / nel[0], 0.2 / nel[1], 0.1 / nel[2]) / fem.p_wave_speed(1e9, 0.25, 1000.0)
    _, iters, _ = run_both(gpu, cfg, 15)
    assert (iters == 2).all()      # no Schwarz data: iterate 2 reproduces iterate 1


def test_zero_steps_and_restart(gpu):
    cfg = I.config("c1")
    subs = gpu.build(cfg)
    gpu.set_ics(cfg, subs)                      # host pointers
    st, it = gpu.run(cfg, subs, n_steps=0)
    assert it.shape[0] == 0
    u_a, _ = gpu.fom_state(subs[0])
    gpu.run(cfg, subs, n_steps=5)
    gpu.set_ics(cfg, subs, device="cuda:0")     # restart from the IC via device pointers
    u_b, _ = gpu.fom_state(subs[0])
    assert np.array_equal(u_a, u_b)


def test_bitwise_repeatable(gpu):
    cfg = I.scaled(I.config("c3"), 8.0)
    outs = []
    for _ in range(2):
        subs = gpu.build(cfg)
        gpu.set_ics(cfg, subs, device="cuda:0")
        gpu.run(cfg, subs, n_steps=6)
        outs.append([gpu.fom_state(s) for s in subs])
    for a, b in zip(*outs):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_invalid_arguments(gpu, c2_ops):
    from paper_2511_20687_b200 import osam
    with pytest.raises(osam.OsamError) as e:
        osam.Subdomain(osam.OSAM_FOM, (0, 0, 0), (1, 1, 1), (0, 2, 2), 1e9, 0.25, 1000.0)
    assert e.value.code == -1
    with pytest.raises(osam.OsamError):
        osam.Subdomain(osam.OSAM_FOM, (0, 0, 0), (-1, 1, 1), (2, 2, 2), 1e9, 0.25, 1000.0)
    cfg = I.config("c2")
    bad = dict(c2_ops[1])
    bad["Phi"] = bad["Phi"][:-3]
    subs = gpu.build(cfg, {1: bad})
    gpu.set_ics(cfg, subs)
    with pytest.raises(osam.OsamError) as e:
        gpu.run(cfg, subs, n_steps=1)
    assert e.value.code == -1
    cfg1 = I.config("c1")
    subs = gpu.build(cfg1)
    gpu.set_ics(cfg1, subs)
    with pytest.raises(osam.OsamError):
        osam.osam_step(subs, -1.0, 1e-10, 1)
    with pytest.raises(osam.OsamError):
        osam.osam_step(subs, cfg1["dt"], 1e-10, 1, min_iters=1)


def test_graph_controller_equals_host_loop_bitwise(gpu):
    """The CUDA-graph controller (device-side while-loop over sweeps) and the host-driven loop of
    profiling mode run the same kernels in the same order: bitwise identical states and counts."""
    from paper_2511_20687_b200 import osam
    cfg = I.scaled(I.config("c3"), 10.0)
    out = []
    for prof in (False, True):
        osam.set_profiling(prof)
        try:
            subs = gpu.build(cfg)
            gpu.set_ics(cfg, subs, device="cuda:0")
            _, it = gpu.run(cfg, subs, n_steps=7)
            out.append((it, [gpu.fom_state(s) for s in subs]))
        finally:
            osam.set_profiling(False)
    assert np.array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("max_iters", [1, 2])
def test_max_iters_reached_keeps_last_iterate(gpu, max_iters):
    """Hitting max_iters returns OSAM_WNOTCONVERGED (1) and keeps the last iterate (reading R9), equal to
    the oracle run with the same cap."""
    cfg = dict(I.config("c1"), max_iters=max_iters)
    subs = gpu.build(cfg)
    gpu.set_ics(cfg, subs, device="cuda:0")
    status, iters = gpu.run(cfg, subs, n_steps=5)
    assert status == 1
    assert (iters == max_iters).all()
    models, states, it_ref, _ = oracle_run(cfg, 5)
    assert np.array_equal(iters, it_ref.reshape(iters.shape))
    compare(gpu, subs, models, states)


@pytest.mark.parametrize("prof", [False, True])
def test_unstable_returns_eunstable(gpu, prof):
    """Tiled K1, graph controller and host-driven loop: dt 40x the stability limit overflows the state and
    osam_step returns OSAM_EUNSTABLE (include/osam.h: non-finite convergence norm)."""
    from paper_2511_20687_b200 import osam
    cfg = I.scaled(I.config("c3"), 10.0)
    cfg = dict(cfg, dt=40.0 * cfg["dt"])
    osam.set_profiling(prof)
    try:
        subs = gpu.build(cfg)
        gpu.set_ics(cfg, subs, device="cuda:0")
        with pytest.raises(osam.OsamError) as e:
            gpu.run(cfg, subs, n_steps=200)
        assert e.value.code == -5
    finally:
        osam.set_profiling(False)


@pytest.mark.parametrize("order", [2, 3])
def test_c2_polynomial_opinf(gpu, order):
    """QOpInf / COpInf (eq:quadratic_opinf): c2's FOM-ROM coupling with a quadratic or cubic
    OpInf ROM trained by the oracle's offline stage (r = 20), 200 steps vs the oracle."""
    cfg = I.config("c2")
    cfg["rom"] = dict(cfg["rom"], order=order)
    ops = opinf.train(cfg, I)
    assert ("Hbar" in ops[1]) and (("Cbar" in ops[1]) == (order == 3))
    _, iters, worst = run_both(gpu, cfg, 200, rom_ops=ops, checkpoints=(1,))
    print(f"c2 order {order} worst rel L2", worst)


def test_c5_shaped_batched_cubic_opinf_tensor_cores(gpu):
    """Batched COpInf on the tensor-core path: c5 geometry and samples (B = 64), r = 10, seeded cubic
    operators whose polynomial terms are of the order of the linear one, 100 steps vs the oracle."""
    cfg = I.config("c5")
    rng = np.random.default_rng(12)
    ops = {}
    from paper_2511_20687_b200 import problem
    for i in (0, 1):
        n_free, n_s = problem.dof_split(cfg, i)
        o = I.synthetic_rom_operators(n_free, n_s, 10, 5, cfg["dt"], seed=40 + i)
        k = np.diag(o["Kbar"]).max()
        o["Hbar"] = 0.1 * k / 1e-3 * rng.standard_normal((10, opinf.n_poly(10, 2))) / 55
        o["Cbar"] = 0.1 * k / 1e-6 * rng.standard_normal((10, opinf.n_poly(10, 3))) / 220
        ops[i] = o
    _, iters, worst = run_both(gpu, cfg, 100, rom_ops=ops, checkpoints=(1,))
    print("c5-shaped cubic worst rel L2", worst)


# ---- NEXT-1: multi-substep controller intervals (Xi) and the implicit ROM ------------------------

def _substeps(cfg, n_sub, integrators=None, dt_factor=1.0):
    import copy
    c = copy.deepcopy(cfg)
    for k, s in enumerate(c["subdomains"]):
        s["n_sub"] = n_sub[k]
        if integrators:
            s["integrator"] = integrators[k]
    c["dt"] = cfg["dt"] * dt_factor
    return c


@pytest.mark.parametrize("n_sub,dt_factor", [((2, 2), 2.0), ((1, 3), 1.5), ((3, 2), 2.0), ((4, 1), 1.0)])
def test_c1_substeps_xi(gpu, n_sub, dt_factor):
    """FOM-FOM with n_i substeps per controller step (three-buffer chain, z-form norm, traces + Xi)."""
    cfg = _substeps(I.config("c1"), n_sub, dt_factor=dt_factor)
    _, iters, worst = run_both(gpu, cfg, 60, checkpoints=(1, 7))
    print("c1", n_sub, "worst rel L2", worst, "iters", np.unique(iters))


def test_rigid_translation_mixed_substeps_gpu(gpu):
    """The oracle pin's free-floating bar (uniform translation, v0 through osam_set_ic) on the GPU:
    parity with the oracle and rigid to rounding."""
    from paper_2511_20687_b200 import osam
    subs_cfg = [I._sub("a", "fom", (0, 0, 0), (0.6, 0.1, 0.1), (30, 5, 5)),
                I._sub("b", "fom", (0.4, 0, 0), (1.0, 0.1, 0.1), (24, 4, 4))]
    subs_cfg[0]["n_sub"], subs_cfg[1]["n_sub"] = 1, 3
    cfg = dict(subdomains=subs_cfg, E=I.E0, nu=I.NU, rho=I.RHO, dt=I._dt(subs_cfg), tol=1e-12, max_iters=50,
               min_iters=2)
    models = schwarz.build_models(cfg)
    c = np.array([1e-3, -2e-3, 5e-4])
    vel = np.array([0.7, -0.3, 1.1])
    u0s = [np.broadcast_to(c, (1, m.box.n_nodes, 3)).copy() for m in models]
    v0s = [np.broadcast_to(vel, (1, m.box.n_nodes, 3)).copy() for m in models]
    states, it_ref = schwarz.run(models, u0s, cfg["dt"], 25, cfg["tol"], 50, 2, v0s=v0s)
    subs = gpu.build(cfg)
    for sub, u0, v0 in zip(subs, u0s, v0s):
        sub.set_ic(gpu.soa(u0), gpu.soa(v0))
    _, it = gpu.run(cfg, subs, n_steps=25)
    assert np.array_equal(it.reshape(-1), it_ref.reshape(-1))
    T = 25 * cfg["dt"]
    for sub, m, st in zip(subs, models, states):
        u, v, a = gpu.fom_state(sub, accel=True)
        assert rel(u, st["u"][0]) <= TOL and rel(v, st["v"][0]) <= TOL
        # a is rounding noise of K (c + v t) on both sides: bound it by the stiffness scale instead
        scale = I.E0 / (I.RHO * m.box.h.min() ** 2) * np.abs(u).max()
        assert np.abs(a).max() <= 1e-12 * scale and np.abs(st["a"]).max() <= 1e-12 * scale
        free = m.codes == fem.FREE
        assert np.abs(np.where(free, u - (c + vel * T), 0)).max() <= 1e-12 * np.abs(vel * T).max()


@pytest.fixture(scope="module")
def c2_linear_ops():
    return opinf.train(I.config("c2"), I)


@pytest.mark.parametrize("n_sub,integ,dt_factor", [
    ((2, 1), ("explicit", "implicit"), 2.0),     # torsion-like pairing: explicit FOM, implicit ROM
    ((1, 1), ("explicit", "implicit"), 1.0),
    ((2, 3), ("explicit", "explicit"), 2.0),
])
def test_c2_implicit_rom_and_substeps(gpu, c2_linear_ops, n_sub, integ, dt_factor):
    cfg = _substeps(I.config("c2"), n_sub, integ, dt_factor)
    _, iters, worst = run_both(gpu, cfg, 150, rom_ops=c2_linear_ops, checkpoints=(1,))
    print("c2", n_sub, integ, "worst rel L2", worst, "iters", np.unique(iters))


@pytest.mark.parametrize("tc", ["1", "0"])
def test_c5_shaped_batched_implicit_and_substeps(gpu, monkeypatch, tc):
    """Batched ROM-ROM (B = 64): implicit ROM (per-sample (I + beta dt^2 e_b Kbar)^-1) coupled to an explicit
    ROM taking 2 substeps; tensor-core and CUDA-core paths; per-sample freezing with traces."""
    monkeypatch.setenv("OSAM_ROM_TC", tc)
    cfg = _substeps(I.config("c5"), (1, 2), ("implicit", "explicit"), 2.0)
    from paper_2511_20687_b200 import problem
    ops = {}
    for i in (0, 1):
        n_free, n_s = problem.dof_split(cfg, i)
        ops[i] = I.synthetic_rom_operators(n_free, n_s, 12, 6, I.config("c5")["dt"], seed=60 + i)
    _, iters, worst = run_both(gpu, cfg, 60, rom_ops=ops, checkpoints=(1,))
    print("c5-shaped implicit/substeps tc", tc, "worst rel L2", worst, "iters", np.unique(iters))


def test_graph_equals_host_controller_with_substeps(gpu):
    """Graph-mode and host-driven controller steps agree bitwise with traces and substeps."""
    from paper_2511_20687_b200 import osam
    cfg = _substeps(I.config("c1"), (3, 2), dt_factor=2.0)
    out = []
    for prof in (False, True):
        osam.set_profiling(prof)
        try:
            subs = gpu.build(cfg)
            gpu.set_ics(cfg, subs)
            _, it = gpu.run(cfg, subs, n_steps=20)
            out.append((it, [gpu.fom_state(s) for s in subs]))
        finally:
            osam.set_profiling(False)
    assert np.array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---- NEXT-3: nonlinear FOM (Saint Venant-Kirchhoff / Neohookean, kernel NL1) ------------------------

def _nonlinear(cfg, material, amplitude=None):
    import copy
    c = copy.deepcopy(cfg)
    c["material"] = material
    if amplitude is not None:
        c["ic"] = dict(c["ic"], A=amplitude)
    return c


@pytest.mark.parametrize("material", ["svk", "neohookean"])
def test_c1_nonlinear_fom(gpu, material):
    """c1 geometry at strains ~1e-1 (IC amplitude 2e-2): NL1 against the oracle's element loop."""
    cfg = _nonlinear(I.config("c1"), material, 2e-2)
    _, iters, worst = run_both(gpu, cfg, 80, checkpoints=(1, 9))
    print("c1", material, "worst rel L2", worst, "iters", np.unique(iters))


def test_c1_svk_with_substeps(gpu):
    cfg = _substeps(_nonlinear(I.config("c1"), "svk", 2e-2), (2, 1), dt_factor=2.0)
    _, iters, worst = run_both(gpu, cfg, 40, checkpoints=(1,))
    print("c1 svk substeps worst rel L2", worst)


@pytest.mark.parametrize("material", ["svk", "neohookean"])
def test_c3_scaled_nonlinear_multi_tile(gpu, material):
    """c3 geometry coarsened 5x: several NL1 tiles in x, y and several z-chunks per subdomain, clamped face."""
    cfg = _nonlinear(I.scaled(I.config("c3"), 5.0), material)
    _, iters, worst = run_both(gpu, cfg, 4, checkpoints=(1,))
    print("c3/5", material, "worst rel L2", worst, "iters", np.unique(iters))


def test_c2_svk_fom_with_copinf_rom(gpu):
    """The pairing the paper uses for cubic nonlinearity: SVK FOM coupled to a COpInf ROM trained
    on SVK single-domain data."""
    cfg = _nonlinear(I.config("c2"), "svk", 1e-2)
    cfg["rom"] = dict(cfg["rom"], order=3)
    ops = opinf.train(cfg, I)
    _, iters, worst = run_both(gpu, cfg, 100, rom_ops=ops, checkpoints=(1,))
    print("c2 svk + COpInf worst rel L2", worst, "iters", np.unique(iters))


def test_c2_implicit_qopinf_rom_with_explicit_fom_substeps(gpu):
    """Torsion's pairing: explicit FOM with 2 substeps + implicit QOpInf ROM over controller step 2 dt
    (Newton per step, reading R37), trained operators."""
    cfg = I.config("c2")
    cfg["rom"] = dict(cfg["rom"], order=2)
    ops = opinf.train(cfg, I)
    cfg = _substeps(cfg, (2, 1), ("explicit", "implicit"), 2.0)
    _, iters, worst = run_both(gpu, cfg, 120, rom_ops=ops, checkpoints=(1,))
    print("c2 implicit QOpInf worst rel L2", worst, "iters", np.unique(iters))


@pytest.mark.parametrize("tc", ["1", "0"])
def test_c5_shaped_batched_implicit_cubic_rom(gpu, monkeypatch, tc):
    monkeypatch.setenv("OSAM_ROM_TC", tc)
    cfg = _substeps(I.config("c5"), (1, 2), ("implicit", "explicit"), 2.0)
    rng = np.random.default_rng(21)
    from paper_2511_20687_b200 import problem
    ops = {}
    for i in (0, 1):
        n_free, n_s = problem.dof_split(cfg, i)
        o = I.synthetic_rom_operators(n_free, n_s, 8, 5, I.config("c5")["dt"], seed=70 + i)
        if i == 0:
            k = np.abs(o["Kbar"]).max()
            o["Hbar"] = 0.02 * k / 1e-3 * rng.standard_normal((8, opinf.n_poly(8, 2))) / 36
            o["Cbar"] = 0.02 * k / 1e-6 * rng.standard_normal((8, opinf.n_poly(8, 3))) / 120
        ops[i] = o
    _, iters, worst = run_both(gpu, cfg, 40, rom_ops=ops, checkpoints=(1,))
    print("c5-shaped implicit cubic tc", tc, "worst rel L2", worst, "iters", np.unique(iters))


def test_xlast_column_excluded_c1_variant(gpu):
    """nx a multiple of the 32-node tile and a Schwarz x+ face: the last node column leaves the tiled grid
    (the xlast CTAs of the tiled launch write its prescribed values)."""
    import copy
    cfg = copy.deepcopy(I.config("c1"))
    cfg["subdomains"][0] = dict(cfg["subdomains"][0], nel=(32, 5, 5))
    cfg["dt"] = I._dt(cfg["subdomains"])
    _, iters, worst = run_both(gpu, cfg, 60, checkpoints=(1,))
    print("c1 nx=32 worst rel L2", worst)


def test_xlast_column_excluded_c4_topology(gpu):
    """c4 coarsened 8x: FOM 32^3 elements between two ROMs (stand-in operators), both FOM x-faces Schwarz."""
    from paper_2511_20687_b200 import problem
    cfg = I.scaled(I.config("c4"), 8.0)
    assert cfg["subdomains"][1]["nel"][0] == 32
    cfg["rom"] = dict(cfg["rom"], r=12)
    ops = problem.synthetic_rom_ops(cfg, r_b=8)
    _, iters, worst = run_both(gpu, cfg, 6, rom_ops=ops, checkpoints=(1,))
    print("c4/8 worst rel L2", worst, "iters", np.unique(iters))
