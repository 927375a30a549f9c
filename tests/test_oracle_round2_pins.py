"""Further oracle pins (SURVEY 8(c) c.3 rows that round 1 left open).

* the C element-loop force (oracle/cfem.c) against the brute-force assembled K, rigid modes and the
  NumPy loop (two independent element loops of the same definition);
* top-down training (oracle.opinf.train_coupled, Algorithm 2 steps 1-2) against SURVEY
  finding 9 (an independent prototype): c5 snapshot numerical rank 561 / 490 at 1e-13 relative and
  r_b = 34 / 35 by the 99.9999% energy rule;
* the convergence reduction (eq:conv_criterion P:L443-467): the oracle's (num, den) against a
  compensated (Neumaier) sum of the same per-DOF terms;
* non-conformal FOM-FOM Schwarz (Algorithm 1 with trilinear Pi) converges to the exact
  d'Alembert solution of the nu = 0 bar (R28) at O(h^2) under refinement.
"""
import math

import numpy as np
import pytest

import osam_inputs as I
from oracle import cfem, exact, fem, opinf, schwarz


def neumaier(xs):
    """Kahan-Babuska-Neumaier compensated sum (independent of numpy's pairwise summation)."""
    s = 0.0
    c = 0.0
    for x in xs:
        t = s + x
        if abs(s) >= abs(x):
            c += (s - t) + x
        else:
            c += (x - t) + s
        s = t
    return s + c


# ---- C element loop -------------------------------------------------------------------------------

@pytest.mark.parametrize("nel,h", [((1, 1, 1), (1.0, 1.0, 1.0)), ((4, 3, 2), (0.3, 0.2, 0.5)),
                                   ((3, 5, 4), (0.01, 0.02, 0.015))])
def test_c_force_equals_bruteforce_assembled_K(nel, h):
    box = fem.Box((0, 0, 0), tuple(n * hh for n, hh in zip(nel, h)), nel)
    Ke = fem.hex8_stiffness(box.h, 1e9, 0.25)
    K = fem.assembled_stiffness(box, Ke)
    u = np.random.default_rng(3).standard_normal((box.n_nodes, 3))
    f_ref = (K @ u.reshape(-1)).reshape(-1, 3)
    f_c = cfem.internal_force_c(box, Ke, u)
    assert np.abs(f_c - f_ref).max() <= 1e-13 * np.abs(f_ref).max()


def test_c_force_rigid_modes_and_numpy_loop():
    box = fem.Box((0.45, 0, 0), (1, 1, 1), (11, 13, 9))
    Ke = fem.hex8_stiffness(box.h, 1e9, 0.25)
    X = box.coords()
    Knorm = np.linalg.norm(Ke.reshape(24, 24), 2)
    for u in (np.tile([1.0, -2.0, 0.5], (box.n_nodes, 1)),
              np.stack([-X[:, 1], X[:, 0], np.zeros(len(X))], axis=1),       # rotation about z
              np.stack([np.zeros(len(X)), -X[:, 2], X[:, 1]], axis=1)):      # rotation about x
        f = cfem.internal_force_c(box, Ke, u)
        assert np.linalg.norm(f) <= 1e-15 * Knorm * np.linalg.norm(u) * 8
    u = np.random.default_rng(4).standard_normal((box.n_nodes, 3))
    f_np = fem.internal_force(box, Ke, u)
    f_c = cfem.internal_force_c(box, Ke, u)
    assert np.abs(f_c - f_np).max() <= 1e-14 * np.abs(f_np).max()
    # deterministic: the 8-colouring fixes every node's summation order
    assert np.array_equal(f_c, cfem.internal_force_c(box, Ke, u))


# ---- top-down training ----------------------------------------------------------------------------

@pytest.mark.slow
def test_train_coupled_c5_rank_and_boundary_rank_match_independent_prototype():
    """SURVEY finding 9: the FOM-FOM snapshot matrices of the c5 meshes (2001 snapshots) have numerical rank
    561 / 490 at 1e-13 relative, and the energy rule gives r_b = 34 / 35.  A dropped column, a wrong snapshot
    index or the wrong Schwarz DOF set changes these counts."""
    cfg = I.config("c5")
    ops = opinf.train_coupled(cfg, I)
    rank = {i: int((o["sigma"] > 1e-13 * o["sigma"][0]).sum()) for i, o in ops.items()}
    assert rank == {0: 561, 1: 490}
    assert {i: o["r_b"] for i, o in ops.items()} == {0: 34, 1: 35}
    assert all(len(o["sigma"]) == 2001 for o in ops.values())        # snapshots 0..2000
    assert {i: o["Phi"].shape[1] for i, o in ops.items()} == {0: 400, 1: 400}


# ---- convergence reduction ------------------------------------------------------------------------

def test_convergence_norm_equals_compensated_sum():
    """num, den of eq:conv_criterion from the oracle's controller equal a Neumaier sum of the per-DOF terms
    (free DOFs, (u - u_prev) + dt (v - v_prev) and u + dt v) to 1e-14."""
    cfg = I.config("c1")
    models = schwarz.build_models(cfg)
    states = [m.init_state(I.initial_displacements(cfg, s)) for m, s in zip(models, cfg["subdomains"])]
    for _ in range(3):
        states, _ = schwarz.controller_step(models, states, cfg["tol"])
    # replay one controller step by hand to get the iterates n = 1, 2 and the oracle's trace
    trace = []
    schwarz.controller_step(models, states, cfg["tol"], trace=trace)
    ckpt = states
    it1, it2 = [], []
    for i, m in enumerate(models):        # iterate 1: sources later in the sweep give their checkpoint
        src = [[it1[j]] * 2 if j < i else [ckpt[j]] * 2 for j in range(len(models))]
        it1.append(m.advance(ckpt[i], m.gather_s(src, models, 1)))
    for i, m in enumerate(models):        # iterate 2
        src = [[it2[j]] * 2 if j < i else [it1[j]] * 2 for j in range(len(models))]
        it2.append(m.advance(ckpt[i], m.gather_s(src, models, 1)))
    nums, dens = [], []
    for m, a, b in zip(models, it2, it1):
        free = (m.codes == fem.FREE)[None]
        d = ((a["u"] - b["u"]) + m.dt * (a["v"] - b["v"]))[free]
        w = (a["u"] + m.dt * a["v"])[free]
        nums += list((d * d).ravel())
        dens += list((w * w).ravel())
    n2, num, den = trace[0]
    assert n2 == 2
    assert math.isclose(num[0], neumaier(nums), rel_tol=1e-14) and math.isclose(den[0], neumaier(dens), rel_tol=1e-14)
    assert math.isclose(neumaier(dens), math.fsum(dens), rel_tol=1e-15)   # the compensated sum itself
    assert trace[1][0] == 3 and trace[1][1][0] == 0.0                      # R6: iterate 3 repeats iterate 2


# ---- non-conformal Schwarz: O(h^2) ----------------------------------------------------------------

def _bar_error(n_per_unit):
    """nu = 0 bar [0, 1] (clamped ends in x, lateral faces free: exactly the 1D bar), IC u_x = f(x) =
    A exp(-((x - 0.5)/0.1)^2), two overlapping FOMs [0, 0.6] and [0.4, 1] with non-matching meshes
    (n and 0.8 n elements per unit length); max nodal error against d'Alembert (R28) at c t = 0.3."""
    A = 1e-3
    f = lambda x: A * np.exp(-((x - 0.5) / 0.1) ** 2)
    n1, n2 = int(round(0.6 * n_per_unit)), int(round(0.6 * 0.8 * n_per_unit))
    subs = [I._sub("o1", "fom", (0, 0, 0), (0.6, 0.1, 0.1), (n1, 1, 1), (I.ROLLER_X, 0, 0, 0, 0, 0)),
            I._sub("o2", "fom", (0.4, 0, 0), (1.0, 0.1, 0.1), (n2, 1, 1), (0, I.ROLLER_X, 0, 0, 0, 0))]
    E, nu, rho = 1e9, 0.0, 1000.0
    c = math.sqrt(E / rho)
    h_min = min(0.6 / n1, 0.6 / n2)
    T = 0.3 / c
    n_steps = int(math.ceil(T / (0.5 * h_min / c)))
    dt = T / n_steps
    cfg = dict(subdomains=subs, E=E, nu=nu, rho=rho, dt=dt)
    models = schwarz.build_models(cfg)
    u0 = []
    for s in subs:
        X = I.node_coords(s["lo"], s["hi"], s["nel"])
        u = np.zeros_like(X)
        u[:, 0] = f(X[:, 0])
        u0.append(u[None])
    states, iters = schwarz.run(models, u0, dt, n_steps, 1e-12)
    err = 0.0
    for m, st in zip(models, states):
        X = m.box.coords()
        err = max(err, np.abs(st["u"][0][:, 0] - exact.dalembert(f, 1.0, c, X[:, 0], T)).max())
    return err / A, iters


def test_nonconformal_schwarz_converges_at_second_order():
    errs = []
    for n in (50, 100, 200):
        e, iters = _bar_error(n)
        assert (iters == 3).all()
        errs.append(e)
    rates = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert all(1.8 <= r <= 2.2 for r in rates), (errs, rates)
    assert errs[-1] < 5e-3
