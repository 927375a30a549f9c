"""GPU parity of the small-subdomain FOM path K1S and of the persistent controller for small all-FOM groups (fom_gather_kernel: every node one 4-lane gather of the
class-table stencil, used below OSAM_GATHER_MAX nodes) against the oracle, on the cases that exercise every
node class, the controller variants and the exchange paths."""
import numpy as np
import pytest

import osam_inputs as I
from test_gpu_parity import _substeps, run_both  # noqa: F401  (shared GPU-vs-oracle driver)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["resident", "persistent", "persistent_grid", "graph"])
def gather_path(monkeypatch, request):
    """K1S everywhere; small all-FOM groups run the cluster-resident controller (default, state in shared
    memory, when it fits), the persistent controller as one thread-block cluster (OSAM_SMALL_RESIDENT=0), as a
    grid-wide cooperative launch (OSAM_SMALL_CLUSTER=0), or the per-step CUDA graph (OSAM_SMALL_PERSIST=0)."""
    monkeypatch.setenv("OSAM_GATHER_MAX", str(1 << 30))
    monkeypatch.setenv("OSAM_SMALL_PERSIST", "0" if request.param == "graph" else "1")
    monkeypatch.setenv("OSAM_SMALL_RESIDENT", "1" if request.param == "resident" else "0")
    monkeypatch.setenv("OSAM_SMALL_CLUSTER", "0" if request.param == "persistent_grid" else "1")
    return request.param


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam, problem
    osam.lib()
    return problem


def test_c1_full_horizon_gather(gpu):
    cfg = I.config("c1")
    _, iters, worst = run_both(gpu, cfg, cfg["n_steps"], checkpoints=(1, 50))
    assert (iters == 3).all()


@pytest.mark.parametrize("factor,steps", [(8.0, 15), (5.3, 8)])
def test_scaled_c3_gather(gpu, factor, steps):
    cfg = I.scaled(I.config("c3"), factor)
    run_both(gpu, cfg, steps, checkpoints=(1,))


@pytest.mark.parametrize("nel", [(1, 1, 1), (3, 2, 5), (40, 9, 3)])
def test_single_fom_degenerate_gather(gpu, nel):
    cfg = I.config("c1")
    s = dict(cfg["subdomains"][0], nel=nel, dirichlet=(I.CLAMP, 0, 0, 0, 0, I.ROLLER_X))
    cfg = dict(cfg, subdomains=[s], dt=I._dt([s]))
    run_both(gpu, cfg, 20, checkpoints=(1,))


@pytest.mark.parametrize("n_sub,dt_factor", [((2, 2), 2.0), ((1, 3), 1.5)])
def test_c1_substeps_gather(gpu, n_sub, dt_factor):
    run_both(gpu, _substeps(I.config("c1"), n_sub, dt_factor=dt_factor), 40, checkpoints=(1,))


def test_graph_equals_host_gather(gpu):
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


def test_c2_fom_rom_gather(gpu):
    from oracle import opinf
    cfg = I.config("c2")
    run_both(gpu, cfg, 150, rom_ops=opinf.train(cfg, I), checkpoints=(1,))


@pytest.mark.parametrize("max_iters", [1, 2])
def test_max_iters_gather(gpu, max_iters):
    """The cap on the small path (both controllers): OSAM_WNOTCONVERGED, the last iterate kept (R9), equal
    to the oracle run with the same cap, over an odd number of steps (the persistent kernel's role swap)."""
    from test_gpu_parity import compare, oracle_run
    cfg = dict(I.config("c1"), max_iters=max_iters)
    subs = gpu.build(cfg)
    gpu.set_ics(cfg, subs, device="cuda:0")
    status, iters = gpu.run(cfg, subs, n_steps=5)
    assert status == 1
    assert (iters == max_iters).all()
    models, states, it_ref, _ = oracle_run(cfg, 5)
    assert np.array_equal(iters, it_ref.reshape(iters.shape))
    compare(gpu, subs, models, states)


def test_unstable_gather(gpu):
    """dt 40x the explicit stability limit: the state overflows within ~100 steps and osam_step returns
    OSAM_EUNSTABLE (non-finite convergence norm) on both controllers."""
    from paper_2511_20687_b200 import osam
    cfg = I.config("c1")
    cfg = dict(cfg, dt=40.0 * cfg["dt"])
    subs = gpu.build(cfg)
    gpu.set_ics(cfg, subs, device="cuda:0")
    with pytest.raises(osam.OsamError) as e:
        gpu.run(cfg, subs, n_steps=200)
    assert e.value.code == -5


def test_controllers_bitwise_c1(gpu, monkeypatch, gather_path):
    """c1 over an odd number of steps: every small-group controller (resident, persistent cluster, persistent
    grid) leaves states bitwise equal to the per-step graph's (same per-node arithmetic) and the same counts."""
    if gather_path != "resident":
        pytest.skip("runs every controller itself")
    cfg = I.config("c1")
    out = {}
    for name, env in (("graph", dict(OSAM_SMALL_PERSIST="0")),
                      ("resident", dict(OSAM_SMALL_PERSIST="1", OSAM_SMALL_RESIDENT="1")),
                      ("persistent", dict(OSAM_SMALL_PERSIST="1", OSAM_SMALL_RESIDENT="0", OSAM_SMALL_CLUSTER="1")),
                      ("grid", dict(OSAM_SMALL_PERSIST="1", OSAM_SMALL_RESIDENT="0", OSAM_SMALL_CLUSTER="0"))):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        subs = gpu.build(cfg)
        gpu.set_ics(cfg, subs, device="cuda:0")
        _, it = gpu.run(cfg, subs, n_steps=37)
        _, it2 = gpu.run(cfg, subs, n_steps=4)  # a second call continues from the written-back state
        out[name] = (np.concatenate([it.ravel(), it2.ravel()]), [gpu.fom_state(s) for s in subs])
    ref = out["graph"]
    for name, (it, st) in out.items():
        assert np.array_equal(it, ref[0]), name
        for a, b in zip(st, ref[1]):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), name
