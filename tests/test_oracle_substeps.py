"""Pins for the oracle's multi-substep controller intervals, the temporal interpolant Xi and the
implicit (average-acceleration) ROM (P:L404-442 eq:schwarz_discrete, L468-490,
L617-722 eq:schwarz_opinf_discrete; readings R31-R33)."""
import copy

import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, schwarz


def _run(cfg, n_steps, v0s=None, tol=None, max_iters=50):
    models = schwarz.build_models(cfg, cfg.get("_ops"), cfg.get("_e"))
    u0s = cfg.get("_u0s") or [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    st, it = schwarz.run(models, u0s, cfg["dt"], n_steps, tol or cfg["tol"], max_iters, 2, v0s=v0s)
    return models, st, it


def _with_substeps(cfg, n_sub, dt=None):
    c = copy.deepcopy(cfg)
    for s, m in zip(c["subdomains"], n_sub):
        s["n_sub"] = m
    if dt is not None:
        c["dt"] = dt
    return c


def test_equal_substeps_equal_finer_controller_steps_bitwise():
    """n_i = 2 on both subdomains over controller step dt  ==  n_i = 1 over dt/2, twice as many steps:
    Xi is the identity on coinciding times and the converged iterates are exact fixed points
    (num == 0, reading R6), so the two runs agree bit for bit."""
    cfg = I.config("c1")
    _, a, ia = _run(_with_substeps(cfg, (2, 2)), 40)
    _, b, ib = _run(_with_substeps(cfg, (1, 1), cfg["dt"] / 2), 80)
    assert (ia == 3).all() and (ib == 3).all()
    for x, y in zip(a, b):
        assert np.array_equal(x["u"], y["u"]) and np.array_equal(x["v"], y["v"]) and np.array_equal(x["a"], y["a"])


def _free_bar(n_sub):
    subs = [I._sub("a", "fom", (0, 0, 0), (0.6, 0.1, 0.1), (30, 5, 5)),
            I._sub("b", "fom", (0.4, 0, 0), (1.0, 0.1, 0.1), (24, 4, 4))]
    for s, m in zip(subs, n_sub):
        s["n_sub"] = m
    return dict(subdomains=subs, E=I.E0, nu=I.NU, rho=I.RHO, dt=I._dt(subs), tol=1e-12)


@pytest.mark.parametrize("n_sub", [(1, 3), (3, 2), (2, 5), (4, 1)])
def test_rigid_translation_exact_with_mixed_substeps(n_sub):
    """A free-floating two-box bar in uniform translation u = c + v t: K annihilates rigid motions, so
    every explicit Newmark substep is exact, and Xi, linear in time, reproduces the donor's motion at any
    destination substep. The coupled run must stay rigid to rounding; a Xi that drops the interpolation
    (nearest earlier donor substep) is off by ~1e-2."""
    cfg = _free_bar(n_sub)
    models = schwarz.build_models(cfg)
    c = np.array([1e-3, -2e-3, 5e-4])
    vel = np.array([0.7, -0.3, 1.1])
    cfg["_u0s"] = [np.broadcast_to(c, (1, m.box.n_nodes, 3)).copy() for m in models]
    v0s = [np.broadcast_to(vel, (1, m.box.n_nodes, 3)).copy() for m in models]
    n = 25
    models, st, it = _run(cfg, n, v0s=v0s)
    T = n * cfg["dt"]
    for m, s in zip(models, st):
        free = m.codes == fem.FREE
        assert np.abs(np.where(free, s["u"][0] - (c + vel * T), 0)).max() <= 1e-12 * np.abs(vel * T).max()
        assert np.abs(np.where(free, s["v"][0] - vel, 0)).max() <= 1e-11 * np.abs(vel).max()


# ---- ROM alone (no Schwarz boundary): closed forms ---------------------------------------------

def _lone_rom(Kbar, dt, n_sub=1, integrator="implicit", e=None, seed=0):
    sub = I._sub("rom", "rom", (0, 0, 0), (1.0, 0.1, 0.1), (20, 2, 2), (I.CLAMP, I.CLAMP, 0, 0, 0, 0))
    sub["n_sub"] = n_sub
    sub["integrator"] = integrator
    cfg = dict(subdomains=[sub], E=I.E0, nu=I.NU, rho=I.RHO, dt=dt, tol=1e-10)
    box = fem.Box(sub["lo"], sub["hi"], sub["nel"])
    n_free = int((fem.dof_codes(box, sub["dirichlet"], []) == fem.FREE).sum())
    r = Kbar.shape[0]
    Phi = np.linalg.qr(np.random.default_rng(seed).standard_normal((n_free, r)))[0]
    ops = {0: dict(Phi=Phi, Phi_s=np.zeros((0, 0)), Kbar=Kbar, Bbar=np.zeros((r, 0)))}
    model = schwarz.build_models(cfg, ops, e)[0]
    u0 = np.zeros((1, box.n_nodes, 3))
    u0.reshape(1, -1)[0, model.free_dofs] = Phi @ np.linspace(1.0, 2.0, r) * 1e-3
    return cfg, model, u0


def _modal(r, seed):
    rng = np.random.default_rng(seed)
    V = np.eye(r) + 0.3 * rng.standard_normal((r, r))
    return V


@pytest.mark.parametrize("n_sub", [1, 2])
def test_implicit_rom_closed_form_nonsymmetric_modes(n_sub):
    """Average acceleration is the trapezoidal rule on (u, v): for u'' = -w^2 u it rotates (u, v/w) by
    theta = 2 atan(w dt/2) per step, at any w dt (unconditionally stable). With Kbar = V diag(w^2) V^-1
    (non-symmetric: a transposed Kbar fails) and per-sample scale e_b (w -> sqrt(e_b) w):
        u^_n = V diag(cos(n theta)) V^-1 u^_0 ,  v^_n = -V diag(w sin(n theta)) V^-1 u^_0."""
    dt_c = 1e-4
    wdt = np.array([0.3, 1.0, 3.0, 10.0])               # per substep; beyond the explicit limit 2
    dt = dt_c / n_sub
    w = wdt / dt
    V = _modal(4, 3)
    Kbar = V @ np.diag(w ** 2) @ np.linalg.inv(V)
    e = np.array([1.0, 0.5, 2.0])
    cfg, model, u0 = _lone_rom(Kbar, dt_c, n_sub, "implicit", e)
    st = model.init_state(u0)
    uh0 = st["uh"][0]
    c0 = np.linalg.solve(V, uh0)
    for k in range(1, 31):
        st, _ = schwarz.controller_step([model], [st], cfg["tol"])
        st = st[0]
        for b, eb in enumerate(e):
            th = 2 * np.arctan(np.sqrt(eb) * w * dt / 2)
            n = k * n_sub
            u_ref = V @ (np.cos(n * th) * c0)
            v_ref = -V @ (np.sqrt(eb) * w * np.sin(n * th) * c0)
            assert np.abs(st["uh"][b] - u_ref).max() <= 1e-11 * np.abs(c0).max() * np.abs(V).max()
            assert np.abs(st["vh"][b] - v_ref).max() <= 1e-11 * np.abs(np.sqrt(eb) * w * c0).max() * np.abs(V).max()


def test_implicit_rom_energy_conserved_spd():
    """Average acceleration conserves 1/2 |v^|^2 + 1/2 u^T Kbar u^ exactly for symmetric Kbar and no
    forcing, even at w dt = 50."""
    rng = np.random.default_rng(9)
    Q = np.linalg.qr(rng.standard_normal((6, 6)))[0]
    dt = 1e-4
    Kbar = Q @ np.diag((np.array([0.1, 0.5, 1, 4, 20, 50]) / dt) ** 2) @ Q.T
    cfg, model, u0 = _lone_rom(Kbar, dt)
    st = model.init_state(u0)
    energy = lambda s: 0.5 * s["vh"][0] @ s["vh"][0] + 0.5 * s["uh"][0] @ Kbar @ s["uh"][0]
    e0 = energy(st)
    for _ in range(200):
        st = schwarz.controller_step([model], [st], cfg["tol"])[0][0]
        assert abs(energy(st) - e0) <= 1e-10 * e0      # rounding only (cond ~ (w dt)^2)


@pytest.mark.parametrize("integrator", ["explicit", "implicit"])
def test_rom_substeps_equal_finer_steps(integrator):
    """A ROM alone with n_i = 3 over dt equals n_i = 1 over dt/3, three times as many steps."""
    V = _modal(5, 4)
    Kbar = V @ np.diag((np.array([0.1, 0.4, 0.8, 1.2, 1.5]) / 1e-4) ** 2) @ np.linalg.inv(V)
    cfg3, m3, u0 = _lone_rom(Kbar, 3e-4, 3, integrator)
    cfg1, m1, _ = _lone_rom(Kbar, 3e-4 / 3, 1, integrator)     # the same dt_i bit for bit
    a, b = m3.init_state(u0), m1.init_state(u0)
    for _ in range(10):
        a = schwarz.controller_step([m3], [a], 1e-10)[0][0]
        for _ in range(3):
            b = schwarz.controller_step([m1], [b], 1e-10)[0][0]
    for k in ("uh", "vh", "ah"):
        assert np.array_equal(a[k], b[k])


def test_implicit_fom_rejected():
    c1 = I.config("c1")
    c1["subdomains"][0]["integrator"] = "implicit"
    with pytest.raises(ValueError):
        schwarz.build_models(c1)


# ---- implicit polynomial ROM (Newton, reading R37) ------------------------------------------------

def _lone_poly_rom(r, dt, order, seed=0, scale=1.0, n_sub=1, e=None):
    """A lone ROM with a mildly nonlinear polynomial operator (H, C sized so the polynomial terms are ~10%
    of the linear one at |u| ~ 1e-3)."""
    rng = np.random.default_rng(seed)
    w = np.linspace(0.5, 3.0, r) / dt
    V = np.eye(r) + 0.2 * rng.standard_normal((r, r))
    Kbar = V @ np.diag(w ** 2) @ np.linalg.inv(V)
    cfg, model, u0 = _lone_rom(Kbar, dt * n_sub, n_sub, "implicit", e, seed)
    ops = {0: dict(Phi=model.Phi, Phi_s=np.zeros((0, 0)), Kbar=Kbar, Bbar=np.zeros((r, 0)))}
    k = np.abs(Kbar).max()
    if order >= 2:
        n2 = r * (r + 1) // 2
        ops[0]["Hbar"] = scale * 0.1 * k / 1e-3 * rng.standard_normal((r, n2)) / n2
    if order >= 3:
        n3 = r * (r + 1) * (r + 2) // 6
        ops[0]["Cbar"] = scale * 0.1 * k / 1e-6 * rng.standard_normal((r, n3)) / n3
    model = schwarz.build_models(cfg, ops, e)[0]
    return cfg, model, u0, ops[0]


def test_implicit_newton_without_polynomial_terms_is_the_linear_solve():
    cfg, lin, u0 = _lone_rom(np.diag([4e6, 9e6, 2.5e7]), 1e-3)
    ops = {0: dict(Phi=lin.Phi, Phi_s=np.zeros((0, 0)), Kbar=lin.Kbar, Bbar=np.zeros((3, 0)), Hbar=np.zeros((3, 6)))}
    newton = schwarz.build_models(cfg, ops)[0]
    a, b = lin.init_state(u0), newton.init_state(u0)
    for _ in range(50):
        a = schwarz.controller_step([lin], [a], 1e-10)[0][0]
        b = schwarz.controller_step([newton], [b], 1e-10)[0][0]
    for k in ("uh", "vh", "ah"):
        assert np.abs(a[k] - b[k]).max() <= 1e-12 * np.abs(a[k]).max()


@pytest.mark.parametrize("order", [2, 3])
def test_implicit_polynomial_step_satisfies_newmark_with_kronecker_accel(order):
    """After every step: u^' = u~ + dt^2/4 a(u^') and v^' = v^ + dt/2 (a^ + a^'), with a evaluated from the full
    symmetric Kronecker tensors rebuilt independently from the compressed H, C."""
    import itertools
    r, dt = 3, 1e-3
    e = np.array([1.0, 0.7])
    cfg, m, u0, ops = _lone_poly_rom(r, dt, order, seed=order, e=e, scale=0.05)
    Hf = np.zeros((r, r * r))
    Cf = np.zeros((r, r ** 3))
    if "Hbar" in ops:
        for q, (i, j) in enumerate([(i, j) for i in range(r) for j in range(i, r)]):
            perms = set(itertools.permutations((i, j)))
            for a, b in perms:
                Hf[:, a * r + b] = ops["Hbar"][:, q] / len(perms)
    if "Cbar" in ops:
        for q, (i, j, l) in enumerate([(i, j, l) for i in range(r) for j in range(i, r) for l in range(j, r)]):
            perms = set(itertools.permutations((i, j, l)))
            for a, b, c in perms:
                Cf[:, (a * r + b) * r + c] = ops["Cbar"][:, q] / len(perms)

    def acc(u, eb):
        return eb * (-ops["Kbar"] @ u - Hf @ np.kron(u, u) - Cf @ np.kron(np.kron(u, u), u))

    st = m.init_state(u0)
    for _ in range(40):
        new = schwarz.controller_step([m], [st], 1e-10)[0][0]
        for b, eb in enumerate(e):
            ut = st["uh"][b] + dt * st["vh"][b] + 0.25 * dt * dt * st["ah"][b]
            a_new = acc(new["uh"][b], eb)
            assert np.abs(new["uh"][b] - (ut + 0.25 * dt * dt * a_new)).max() <= 1e-13 * np.abs(new["uh"][b]).max()
            assert np.abs(new["ah"][b] - a_new).max() <= 1e-9 * np.abs(a_new).max()
            v_ref = st["vh"][b] + 0.5 * dt * (st["ah"][b] + a_new)
            assert np.abs(new["vh"][b] - v_ref).max() <= 1e-9 * np.abs(v_ref).max()
        assert np.abs(new["uh"]).max() < 10 * np.abs(m.init_state(u0)["uh"]).max()   # a bounded trajectory
        st = new


def test_implicit_polynomial_second_order_against_solve_ivp():
    """Average acceleration is second order: against scipy's DOP853 (rtol 1e-12) on the same cubic ROM ODE,
    the error at T falls by ~4 when dt halves."""
    from scipy.integrate import solve_ivp
    r, T = 2, 2e-2
    errs = []
    for n in (200, 400):
        dt = T / n
        cfg, m, u0, ops = _lone_poly_rom(r, T / 4, 3, seed=11, scale=0.05)    # w dt <= 0.06 at n = 200
        m.dt = dt
        st = m.init_state(u0)
        for _ in range(n):
            st = schwarz.controller_step([m], [st], 1e-10)[0][0]
        y0 = np.concatenate([m.init_state(u0)["uh"][0], np.zeros(r)])
        f = lambda t, y: np.concatenate([y[r:], m.accel(y[None, :r], np.zeros((1, 0)))[0]])
        ref = solve_ivp(f, (0, T), y0, method="DOP853", rtol=1e-12, atol=1e-18).y[:r, -1]
        errs.append(np.abs(st["uh"][0] - ref).max() / np.abs(ref).max())
    assert 3.5 < errs[0] / errs[1] < 4.5, errs
