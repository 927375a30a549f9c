"""Pins for oracle/fem.py against closed forms, brute force and invariants."""
import json
import os

import numpy as np
import pytest

from oracle import exact, fem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rng(seed=0):
    return np.random.default_rng(seed)


def _1d(h):
    """1D linear-element matrices on one element of length h, computed by hand:
    M = int phi_a phi_b, S = int phi_a' phi_b', G = int phi_a' phi_b."""
    M = h / 6.0 * np.array([[2.0, 1.0], [1.0, 2.0]])
    S = 1.0 / h * np.array([[1.0, -1.0], [-1.0, 1.0]])
    G = 0.5 * np.array([[-1.0, -1.0], [1.0, 1.0]])
    return M, S, G


def closed_form_hex8(h, E, nu):
    """Rectangular hex8 stiffness from 1D tensor products (exact integration):
    K[a c, b d] = sum_{j,l} C_cjdl prod_axis m_axis, with m = S on axis j=l, G on j, G^T on l, M else."""
    lam, mu = fem.lame(E, nu)
    C = fem.elasticity_tensor(lam, mu)
    mats = [_1d(hd) for hd in h]
    bits = ((fem.LOCAL_NODES + 1) // 2).astype(int)
    K = np.zeros((8, 3, 8, 3))
    for a in range(8):
        for b in range(8):
            for j in range(3):
                for l in range(3):
                    val = 1.0
                    for ax in range(3):
                        M, S, G = mats[ax]
                        pa, pb = bits[a, ax], bits[b, ax]
                        if ax == j and ax == l:
                            val *= S[pa, pb]
                        elif ax == j:
                            val *= G[pa, pb]
                        elif ax == l:
                            val *= G[pb, pa]
                        else:
                            val *= M[pa, pb]
                    K[a, :, b, :] += C[:, j, :, l] * val
    return K


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (0.02, 0.03, 0.05), (0.55 / 141, 1 / 256, 1 / 256)])
def test_ke_matches_closed_form(h):
    Ke = fem.hex8_stiffness(h, 1e9, 0.25)
    Kc = closed_form_hex8(h, 1e9, 0.25)
    assert np.abs(Ke - Kc).max() <= 1e-13 * np.abs(Kc).max()


def test_ke_unit_cube_diagonal():
    # (lambda + 4 mu)/9 for the unit cube: S*M*M = 1*(1/3)(1/3) per Laplacian term
    E, nu = 1e9, 0.25
    lam, mu = fem.lame(E, nu)
    Ke = fem.hex8_stiffness((1, 1, 1), E, nu)
    assert np.allclose(np.diagonal(Ke.reshape(24, 24)), (lam + 4 * mu) / 9.0, rtol=1e-14)


def test_ke_symmetric_psd_six_rigid_modes():
    Ke = fem.hex8_stiffness((0.02, 0.03, 0.05), 1e9, 0.25).reshape(24, 24)
    assert np.abs(Ke - Ke.T).max() <= 1e-14 * np.abs(Ke).max()
    w = np.linalg.eigvalsh(Ke)
    assert np.sum(np.abs(w) < 1e-10 * w.max()) == 6
    assert w.min() > -1e-10 * w.max()


def test_element_loop_equals_assembled_K():
    box = fem.Box((0, 0, 0), (0.4, 0.9, 0.2), (4, 3, 2))
    Ke = fem.hex8_stiffness(box.h, 1e9, 0.3)
    K = fem.assembled_stiffness(box, Ke)
    u = _rng(1).standard_normal((box.n_nodes, 3))
    f = fem.internal_force(box, Ke, u)
    ref = (K @ u.reshape(-1)).reshape(-1, 3)
    assert np.linalg.norm(f - ref) <= 1e-14 * np.linalg.norm(ref)
    # per-node local version agrees too
    nodes = np.array([0, 7, box.n_nodes // 2, box.n_nodes - 1])
    fl = fem.internal_force_at(box, Ke, lambda ids: u[ids], nodes)
    assert np.abs(fl - ref[nodes]).max() <= 1e-14 * np.abs(ref).max()


def test_rigid_body_modes_zero_force():
    box = fem.Box((0.1, -0.2, 0.3), (0.7, 0.4, 0.5), (6, 5, 3))
    Ke = fem.hex8_stiffness(box.h, 1e9, 0.25)
    K = fem.assembled_stiffness(box, Ke)
    X = box.coords()
    modes = [np.tile(e, (box.n_nodes, 1)) for e in np.eye(3)]
    for ax in range(3):
        w = np.zeros(3)
        w[ax] = 1.0
        modes.append(np.cross(w[None, :], X))
    nK = np.linalg.norm(K, 2)
    for u in modes:
        f = fem.internal_force(box, Ke, u)
        assert np.linalg.norm(f) <= 1e-15 * nK * np.linalg.norm(u)


def test_patch_test_uniform_strain():
    """u = eps0 X: interior forces vanish; boundary forces = int_dOmega N_a sigma0 n dS."""
    box = fem.Box((0, 0, 0), (0.4, 0.9, 0.2), (4, 3, 2))
    E, nu = 1e9, 0.25
    lam, mu = fem.lame(E, nu)
    Ke = fem.hex8_stiffness(box.h, E, nu)
    eps = np.array([[1.0, 0.3, -0.2], [0.3, -0.5, 0.1], [-0.2, 0.1, 0.7]]) * 1e-3
    sig = lam * np.trace(eps) * np.eye(3) + 2 * mu * eps
    X = box.coords()
    u = X @ eps.T
    f = fem.internal_force(box, Ke, u)
    expect = np.zeros_like(f)
    h = box.h
    for face in range(6):
        ax, side = face // 2, face % 2
        n = np.zeros(3)
        n[ax] = 1.0 if side else -1.0
        o = [d for d in range(3) if d != ax]
        nodes = box.face_nodes(face)
        ijk = np.stack(box.ijk(nodes), axis=1)
        # nodal tributary area: h_e h_f, halved on each face edge
        area = np.ones(len(nodes)) * h[o[0]] * h[o[1]]
        for d in o:
            area *= np.where((ijk[:, d] == 0) | (ijk[:, d] == box.nel[d]), 0.5, 1.0)
        expect[nodes] += area[:, None] * (sig @ n)[None, :]
    assert np.abs(f - expect).max() <= 1e-12 * np.abs(expect).max()


def test_lumped_mass_closed_form():
    m = fem.hex8_lumped_mass((1, 1, 1), 1000.0)
    assert np.allclose(m, 125.0, rtol=1e-15)          # S:L169 example
    box = fem.Box((0, 0, 0), (0.6, 0.1, 0.1), (30, 5, 5))
    ml = fem.lumped_mass(box, 1000.0)
    assert abs(ml.sum() - 1000.0 * 0.6 * 0.1 * 0.1) <= 1e-12 * ml.sum()
    i, j, k = box.ijk(np.arange(box.n_nodes))
    nint = ((i > 0) & (i < 30)).astype(int) + 1
    nint *= ((j > 0) & (j < 5)).astype(int) + 1
    nint *= ((k > 0) & (k < 5)).astype(int) + 1
    assert np.allclose(ml, 1000.0 * np.prod(box.h) / 8 * nint, rtol=1e-14)


def test_cfl_paper_value():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["cfl_1d_wave"]
    c = fem.p_wave_speed(g["E"], g["nu"], g["rho"])     # nu = 0: c_p = sqrt(E/rho)
    assert abs(g["dz"] / c - g["dt"]) <= 1e-15


def _bar(nx=200, L=1.0, E=1e9, rho=1000.0):
    box = fem.Box((0, 0, 0), (L, L / nx, L / nx), (nx, 1, 1))
    # lateral rollers (y faces hold u_y, z faces hold u_z), clamped ends hold u_x
    dirichlet = (1, 1, 2, 2, 4, 4)
    return box, dirichlet


def test_nu0_reduces_to_1d_bar():
    box, _ = _bar(40)
    Ke = fem.hex8_stiffness(box.h, 1e9, 0.0)
    x = box.coords()[:, 0]
    u = np.zeros((box.n_nodes, 3))
    u[:, 0] = np.sin(3 * x) + x ** 2
    f = fem.internal_force(box, Ke, u)
    assert np.abs(f[:, 1:]).max() <= 1e-14 * np.abs(f).max()
    # 1D lumped FE bar: f_j = (E A/h)(2u_j - u_{j-1} - u_{j+1}) on interior stations, A/4 per node
    h = box.h[0]
    A4 = box.h[1] * box.h[2] / 4
    i, _, _ = box.ijk(np.arange(box.n_nodes))
    inner = (i > 0) & (i < box.nel[0])
    up = u[:, 0]
    f1d = np.zeros(box.n_nodes)
    idx = np.nonzero(inner)[0]
    f1d[idx] = 1e9 * A4 / h * (2 * up[idx] - up[idx - 1] - up[idx + 1])
    assert np.abs(f[inner, 0] - f1d[inner]).max() <= 1e-12 * np.abs(f1d).max()


def test_explicit_newmark_dalembert_courant1():
    """nu=0, 1-element section, lateral rollers, clamped ends, Courant 1 -> nodal d'Alembert (R28)."""
    nx, L, E, rho = 200, 1.0, 1e9, 1000.0
    box, dirichlet = _bar(nx, L, E, rho)
    Ke = fem.hex8_stiffness(box.h, E, 0.0)
    m = fem.lumped_mass(box, rho)
    codes = fem.dof_codes(box, dirichlet, [])
    c = np.sqrt(E / rho)
    dt = box.h[0] / c
    f1 = lambda x: 1e-3 * np.exp(-((x - 0.4) ** 2) / (2 * 0.03 ** 2))
    x = box.coords()[:, 0]
    u = np.zeros((box.n_nodes, 3))
    u[:, 0] = f1(x)
    u[codes == fem.DIRICHLET] = 0.0
    force = lambda w: fem.internal_force(box, Ke, w)
    a = np.where(codes == fem.FREE, -force(u) / m[:, None], 0.0)
    v = np.zeros_like(u)
    sd = np.zeros(0, dtype=np.int64)
    worst = 0.0
    for n in range(1, 401):
        u, v, a = fem.explicit_newmark_step(u, v, a, np.zeros(0), codes, sd, force, m, dt)
        ref = exact.dalembert(f1, L, c, x, n * dt)
        worst = max(worst, np.abs(u[:, 0] - ref).max() / 1e-3)
    assert worst <= 1e-12


def test_discrete_energy_conserved():
    """1/2 vbar^T M vbar + 1/2 u^n K u^{n+1} is exactly conserved by central differences."""
    box = fem.Box((0, 0, 0), (1.0, 0.1, 0.1), (50, 5, 5))
    E, nu, rho = 1e9, 0.25, 1000.0
    Ke = fem.hex8_stiffness(box.h, E, nu)
    m = fem.lumped_mass(box, rho)
    codes = fem.dof_codes(box, (1, 1, 0, 0, 0, 0), [])
    dt = 0.5 * box.h.min() / fem.p_wave_speed(E, nu, rho)
    force = lambda w: fem.internal_force(box, Ke, w)
    x = box.coords()[:, 0]
    u = np.zeros((box.n_nodes, 3))
    u[:, 0] = 1e-3 * np.exp(-((x - 0.5) / 0.05) ** 2)
    u[codes == fem.DIRICHLET] = 0
    a = np.where(codes == fem.FREE, -force(u) / m[:, None], 0.0)
    v = np.zeros_like(u)
    sd = np.zeros(0, dtype=np.int64)
    energies = []
    for n in range(600):
        un, vn, an = fem.explicit_newmark_step(u, v, a, np.zeros(0), codes, sd, force, m, dt)
        vbar = (un - u) / dt
        energies.append(0.5 * np.sum(m[:, None] * vbar ** 2) + 0.5 * np.sum(u * force(un)))
        u, v, a = un, vn, an
    e = np.array(energies)
    assert np.abs(e - e[0]).max() <= 1e-12 * e[0]


def test_stability_limit():
    """Central differences are stable iff dt < 2/omega_max (omega_max^2 = lambda_max(M^-1 K)):
    a run at 1.05 dt_crit grows without bound, one at 0.95 dt_crit stays bounded; the configs'
    dt = 0.5 h/c_p (reading R4) sits below dt_crit."""
    box = fem.Box((0, 0, 0), (0.3, 0.06, 0.06), (15, 3, 3))
    E, nu, rho = 1e9, 0.25, 1000.0
    Ke = fem.hex8_stiffness(box.h, E, nu)
    m = fem.lumped_mass(box, rho)
    K = fem.assembled_stiffness(box, Ke)
    Minv = np.repeat(1.0 / m, 3)
    A = Minv[:, None] * K
    w = np.linalg.eigvals(A).real
    lam_max = w.max()
    gersh = np.abs(A).sum(axis=1).max()
    assert lam_max <= gersh * (1 + 1e-12)
    cp, h = fem.p_wave_speed(E, nu, rho), box.h[0]
    dt_crit = 2.0 / np.sqrt(lam_max)
    assert dt_crit > 1.9 * (0.5 * h / cp)
    codes = fem.dof_codes(box, (0,) * 6, [])
    force = lambda u: fem.internal_force(box, Ke, u)
    sd = np.zeros(0, dtype=np.int64)
    growth = {}
    for fac in (0.95, 1.05):
        u = _rng(5).standard_normal((box.n_nodes, 3)) * 1e-6
        a = -force(u) / m[:, None]
        v = np.zeros_like(u)
        n0 = np.linalg.norm(u)
        for _ in range(600):
            u, v, a = fem.explicit_newmark_step(u, v, a, np.zeros(0), codes, sd, force, m, fac * dt_crit)
        growth[fac] = np.linalg.norm(u) / n0
    assert growth[0.95] < 10.0
    assert growth[1.05] > 1e6
