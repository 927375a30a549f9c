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


def test_implicit_polynomial_and_implicit_fom_rejected():
    cfg, model, _ = _lone_rom(np.eye(2) * 1e6, 1e-4)
    n_free, r = len(model.free_dofs), 2
    ops = {0: dict(Phi=np.zeros((n_free, r)), Phi_s=np.zeros((0, 0)), Kbar=np.eye(r), Bbar=np.zeros((r, 0)),
                   Hbar=np.zeros((r, 3)))}
    with pytest.raises(ValueError):
        schwarz.build_models(cfg, ops)
    c1 = I.config("c1")
    c1["subdomains"][0]["integrator"] = "implicit"
    with pytest.raises(ValueError):
        schwarz.build_models(c1)
