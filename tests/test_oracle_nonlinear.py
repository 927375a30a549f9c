"""Pins for the oracle's nonlinear FOM materials (App. A.2, A.3; readings
R35, R36): Saint Venant-Kirchhoff and Neohookean internal forces of the hex8 weak form."""
import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, schwarz

E, NU, RHO = 1e9, 0.25, 1000.0
LAM, MU = fem.lame(E, NU)
KAPPA = LAM + 2 * MU / 3


def _box():
    return fem.Box((0.1, -0.2, 0.3), (0.5, 0.1, 0.55), (4, 3, 5))


def _pk1(material):
    return fem.material_pk1(material, E, NU)


def _random_u(box, scale, seed=0):
    return scale * np.random.default_rng(seed).standard_normal((box.n_nodes, 3))


@pytest.mark.parametrize("material", ["svk", "neohookean"])
def test_small_strain_limit_is_linear_elasticity(material):
    """f(eps u)/eps -> K_e-assembled linear force as eps -> 0, with an O(eps) remainder."""
    box = _box()
    u = _random_u(box, 1.0)
    Ke = fem.hex8_stiffness(box.h, E, NU)
    fl = fem.internal_force(box, Ke, u)
    d = []
    for eps in (1e-5, 5e-6):
        fn = fem.internal_force_nonlinear(box, eps * u, _pk1(material)) / eps
        d.append(np.abs(fn - fl).max() / np.abs(fl).max())
    assert d[0] < 1e-3 and 1.8 < d[0] / d[1] < 2.2


@pytest.mark.parametrize("material", ["svk", "neohookean"])
def test_finite_rigid_rotation_is_stress_free(material):
    """u = (R - I) X + c for a 40-degree rotation: frame indifference gives f = 0 (linear elasticity does not)."""
    box = _box()
    X = box.coords()
    ax = np.array([1.0, 2.0, -0.5]) / np.linalg.norm([1.0, 2.0, -0.5])
    th = np.deg2rad(40.0)
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
    u = X @ (R - np.eye(3)).T + np.array([0.01, -0.02, 0.03])
    scale = E * np.prod(box.h) / box.h.min()          # force of a unit strain on one element
    f = fem.internal_force_nonlinear(box, u, _pk1(material))
    assert np.abs(f).max() <= 1e-12 * scale
    fl = fem.internal_force(box, fem.hex8_stiffness(box.h, E, NU), u)
    assert np.abs(fl).max() > 1e-2 * scale


def _energy_density(material, F):
    """Helmholtz energies as printed: A.2 eq:svk_W (with E = 1/2 (F^T F - I)), A.3 eq:Avol + eq:Adev."""
    C = F.T @ F
    if material == "svk":
        Eg = 0.5 * (C - np.eye(3))
        return 0.5 * LAM * np.trace(Eg) ** 2 + MU * np.trace(Eg @ Eg)
    J2 = np.linalg.det(C)
    return 0.25 * KAPPA * (J2 - np.log(J2) - 1.0) + 0.5 * MU * (J2 ** (-1.0 / 3.0) * np.trace(C) - 3.0)


def _total_energy(material, box, u):
    """W(u) = sum_e sum_q detJ A(F_q), by an explicit per-element, per-point loop."""
    detJ = np.prod(box.h) / 8.0
    W = 0.0
    for ek in range(box.nel[2]):
        for ej in range(box.nel[1]):
            for ei in range(box.nel[0]):
                nodes = [box.node_id(ei + (1 if s[0] > 0 else 0), ej + (1 if s[1] > 0 else 0),
                                     ek + (1 if s[2] > 0 else 0)) for s in fem.LOCAL_NODES]
                ue = u[nodes]
                for q in fem.gauss_points():
                    _, dNdxi = fem.shape_functions(q)
                    dNdX = dNdxi / (box.h / 2.0)
                    F = np.eye(3) + ue.T @ dNdX
                    W += detJ * _energy_density(material, F)
    return W


@pytest.mark.parametrize("material", ["svk", "neohookean"])
def test_force_is_energy_gradient(material):
    """f = dW/du (P = dA/dF, A.2/A.3): central finite differences of the printed energies at strains ~3e-2."""
    box = fem.Box((0, 0, 0), (0.2, 0.1, 0.15), (2, 1, 2))
    u = _random_u(box, 1.5e-3, seed=3)
    f = fem.internal_force_nonlinear(box, u, _pk1(material))
    rng = np.random.default_rng(4)
    dofs = rng.choice(3 * box.n_nodes, 8, replace=False)
    h = 1e-7
    for dof in dofs:
        up, um = u.copy(), u.copy()
        up.reshape(-1)[dof] += h
        um.reshape(-1)[dof] -= h
        fd = (_total_energy(material, box, up) - _total_energy(material, box, um)) / (2 * h)
        assert abs(fd - f.reshape(-1)[dof]) <= 1e-5 * np.abs(f).max()


def test_svk_force_is_cubic_in_the_displacement_scale():
    """A.2: the SVK internal force is a cubic polynomial in s for u -> s u (fourth differences vanish);
    the Neohookean one is not."""
    box = _box()
    u = _random_u(box, 2e-3, seed=7)
    for material, cubic in (("svk", True), ("neohookean", False)):
        g = [fem.internal_force_nonlinear(box, s * u, _pk1(material)) for s in (0.0, 1.0, 2.0, 3.0, 4.0)]
        d4 = g[4] - 4 * g[3] + 6 * g[2] - 4 * g[1] + g[0]
        rel = np.abs(d4).max() / np.abs(g[4]).max()
        assert (rel < 1e-12) if cubic else (rel > 1e-9)


@pytest.mark.parametrize("material", ["svk", "neohookean"])
def test_patch_test_homogeneous_deformation(material):
    """u = (F0 - I) X: uniform stress, so interior nodal forces vanish; boundary forces = P0 N x tributary area."""
    box = _box()
    F0 = np.array([[1.03, 0.02, -0.01], [0.01, 0.98, 0.015], [-0.02, 0.01, 1.01]])
    u = box.coords() @ (F0 - np.eye(3)).T
    f = fem.internal_force_nonlinear(box, u, _pk1(material))
    P0 = _pk1(material)(F0)
    i, j, k = box.ijk(np.arange(box.n_nodes))
    interior = (i > 0) & (i < box.nel[0]) & (j > 0) & (j < box.nel[1]) & (k > 0) & (k < box.nel[2])
    scale = np.abs(P0).max() * box.h[1] * box.h[2]
    assert np.abs(f[interior]).max() <= 1e-10 * scale
    # a node in the interior of face x+ : f = P0 e_x * h_y h_z
    p = box.node_id(box.nel[0], 1, 2)
    assert np.allclose(f[p], P0[:, 0] * box.h[1] * box.h[2], rtol=1e-10, atol=1e-10 * scale)


def test_conformal_fom_fom_svk_equals_monolithic():
    """Conformal SVK FOM-FOM O-SAM equals the single-domain SVK FOM on the union (as for linear elasticity):
    the Schwarz fixed point reproduces the monolithic explicit step exactly, so both runs agree to rounding."""
    cfg = I.config("c1")
    cfg["material"] = "svk"
    cfg["subdomains"][1] = dict(cfg["subdomains"][1], nel=(30, 5, 5))
    cfg["dt"] = 0.5 * 0.02 / fem.p_wave_speed(1e9, 0.25, 1000.0)
    cfg["ic"] = dict(cfg["ic"], A=2e-2)                   # strains ~ 1e-1: strongly nonlinear
    n = 120

    def run(c):
        models = schwarz.build_models(c)
        u0s = [I.initial_displacements(c, s) for s in c["subdomains"]]
        return models, schwarz.run(models, u0s, c["dt"], n, 1e-12, 50, 2)[0]

    models, states = run(cfg)
    mono = dict(cfg, subdomains=[I._sub("mono", "fom", (0, 0, 0), (1, 0.1, 0.1), (50, 5, 5),
                                        (I.ROLLER_X, I.ROLLER_X, 0, 0, 0, 0))])
    mm, ms = run(mono)
    assert mm[0].material == "svk"
    Ym = mm[0].box.coords()
    lin = dict(cfg, material="linear")
    _, ls = run(lin)
    for m, st, sl in zip(models, states, ls):
        X = m.box.coords()
        idx = np.array([np.argmin(np.abs(Ym - x).sum(axis=1)) for x in X])
        ref = ms[0]["u"][0][idx]
        assert np.abs(st["u"][0] - ref).max() <= 1e-9 * np.abs(ref).max()
        assert np.abs(sl["u"][0] - ref).max() > 1e-4 * np.abs(ref).max()    # the nonlinearity matters here
