"""Pins for oracle/opinf.py and the oracle ROM."""
import json
import os

import itertools

import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, opinf, schwarz

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_pod_orthonormal_and_eckart_young():
    rng = np.random.default_rng(0)
    U = rng.standard_normal((300, 40)) @ np.diag(0.7 ** np.arange(40)) @ rng.standard_normal((40, 60))
    r = 7
    Phi, sigma = opinf.pod(U, r)
    assert np.abs(Phi.T @ Phi - np.eye(r)).max() < 1e-12
    resid = np.linalg.norm(U - Phi @ (Phi.T @ U), "fro") ** 2
    assert abs(resid - np.sum(sigma[r:] ** 2)) <= 1e-10 * np.sum(sigma ** 2)
    # optimality (eq:pod_cutoff): no other rank-r orthonormal basis does better
    for s in range(5):
        Q, _ = np.linalg.qr(np.random.default_rng(s + 1).standard_normal((300, r)))
        assert np.linalg.norm(U - Q @ (Q.T @ U), "fro") ** 2 >= resid
    # sign convention R17
    idx = np.argmax(np.abs(Phi), axis=0)
    assert (Phi[idx, np.arange(r)] > 0).all()


def test_energy_rank_by_hand():
    # E_1 = 1/(1 + 1e-6 + 1e-8) < 0.999999 ; E_2 = (1 + 1e-6)/(1 + 1e-6 + 1e-8) >= 0.999999
    assert opinf.energy_rank([1.0, 1e-3, 1e-4]) == 2
    assert opinf.energy_rank([1.0, 1e-4, 1e-4]) == 1
    assert opinf.energy_rank([1.0, 1.0, 1.0, 1.0], 0.5) == 2
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["pod_energy_delta"]
    assert g["delta"] == 0.999999


def test_lambda_grid_paper():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["lambda_grid"]
    n = g["n"]
    grid = 1e-4 * 10.0 ** (4.0 / (n - 1) * np.arange(n))
    assert abs(grid[0] - g["first"]) < 1e-18 and abs(grid[-1] - g["last"]) < 1e-12


def _tiny_fom():
    sub = I._sub("tiny", "fom", (0, 0, 0), (0.1, 0.1, 0.1), (2, 2, 2), (1, 0, 0, 0, 0, 0))
    dt = 0.5 * 0.05 / fem.p_wave_speed(1e9, 0.25, 1000.0)
    return schwarz.FOM(sub, {1: 0}, 1e9, 0.25, 1000.0, dt), dt


def intrusive_operators(m):
    K = fem.assembled_stiffness(m.box, m.Ke)
    Minv = np.repeat(1.0 / m.m, 3)
    Kff = K[np.ix_(m.free_dofs, m.free_dofs)]
    Kfs = K[np.ix_(m.free_dofs, m.schwarz_dofs)]
    return Minv[m.free_dofs, None] * Kff, -Minv[m.free_dofs, None] * Kfs


def test_opinf_recovers_intrusive_operators():
    """Phi = I, lambda = 0, random IC and random Schwarz data -> Kbar = M^-1 K_ff, Bbar = -M^-1 K_fs
    (OpInf consistency P:L278-285)."""
    m, dt = _tiny_fom()
    Kbar_ref, Bbar_ref = intrusive_operators(m)
    rng = np.random.default_rng(7)
    u0 = 1e-3 * rng.standard_normal((1, m.box.n_nodes, 3))
    st = m.init_state(u0)
    nf, ns = len(m.free_dofs), len(m.schwarz_dofs)
    snaps_u, snaps_s = [], []
    for k in range(3 * (nf + ns)):
        s = 1e-3 * rng.standard_normal((1, ns))
        st = m.advance(st, s)
        snaps_u.append(st["u"][0].reshape(-1)[m.free_dofs])
        snaps_s.append(st["u"][0].reshape(-1)[m.schwarz_dofs])
    U = np.stack(snaps_u, 1)
    S = np.stack(snaps_s, 1)
    Kbar, Bbar = opinf.opinf_fit(U, S, dt, 0.0)
    assert np.linalg.norm(Kbar - Kbar_ref) <= 1e-9 * np.linalg.norm(Kbar_ref)
    assert np.linalg.norm(Bbar - Bbar_ref) <= 1e-9 * np.linalg.norm(Bbar_ref)


def test_full_rank_rom_equals_fom():
    """Phi = I, Phi_dS = I, intrusive Kbar, Bbar: a FOM-ROM O-SAM run equals FOM-FOM."""
    cfg = I.config("c1")
    fom_models = schwarz.build_models(cfg)
    m2 = fom_models[1]
    Kbar, Bbar = intrusive_operators(m2)
    ops = {1: dict(Phi=np.eye(len(m2.free_dofs)), Phi_s=np.eye(len(m2.schwarz_dofs)), Kbar=Kbar, Bbar=Bbar)}
    cfg_rom = dict(cfg, subdomains=[cfg["subdomains"][0], dict(cfg["subdomains"][1], kind="rom")])
    rom_models = schwarz.build_models(cfg_rom, rom_ops=ops)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    sf, it_f = schwarz.run(fom_models, u0s, cfg["dt"], 60, cfg["tol"])
    sr, it_r = schwarz.run(rom_models, u0s, cfg["dt"], 60, cfg["tol"])
    assert (it_f == 3).all() and (it_r == 3).all()
    assert np.linalg.norm(sr[0]["u"] - sf[0]["u"]) <= 1e-11 * np.linalg.norm(sf[0]["u"])
    u_rom = rom_models[1].full_field(sr[1])[0]
    free = m2.codes == fem.FREE
    assert np.linalg.norm((u_rom - sf[1]["u"][0])[free]) <= 1e-11 * np.linalg.norm(sf[1]["u"][0][free])


@pytest.fixture(scope="module")
def c2_ops():
    return opinf.train(I.config("c2"), I)


def test_c2_offline_matches_independent_prototype(c2_ops):
    g = json.load(open(os.path.join(GOLD, "survey_crosscheck.json")))["c2"]["offline"]
    o = c2_ops[1]
    assert o["Phi"].shape == (g["N_free"], 20)
    assert o["r_b"] == g["r_b"]
    assert np.isclose(o["sigma"][0], g["sigma1"], rtol=1e-10)
    assert np.isclose(o["sigma"][19] / o["sigma"][0], g["sigma20_over_sigma1"], rtol=1e-6)
    # the prototype solved the ridge through the normal equations; we use augmented LS
    assert np.isclose(np.linalg.norm(o["Kbar"]), g["Kbar_fro"], rtol=1e-8)
    assert np.isclose(np.linalg.norm(o["Bbar"]), g["Bbar_fro"], rtol=1e-8)


def test_c2_online_matches_independent_prototype(c2_ops):
    g = json.load(open(os.path.join(GOLD, "survey_crosscheck.json")))["c2"]
    cfg = I.config("c2")
    models = schwarz.build_models(cfg, rom_ops=c2_ops)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    got = {}

    def cb(k, st):
        if k in (0, 99):
            got[k] = [np.linalg.norm(st[0]["u"]), np.linalg.norm(st[0]["v"]),
                      np.linalg.norm(st[1]["uh"]), np.linalg.norm(st[1]["vh"])]
    _, iters = schwarz.run(models, u0s, cfg["dt"], 100, cfg["tol"], callback=cb)
    assert (iters == 3).all()
    assert np.allclose(got[0], g["after_step_1"], rtol=1e-10)
    assert np.allclose(got[99], g["after_step_100"], rtol=g["rel_tol_100"])


# ---- QOpInf / COpInf (P:L263-272 eq:quadratic_opinf; compressed powers P:L167 footnote) -----------------

def test_khatri_rao_hand_expansions():
    """u = (1, 2) -> (1, 2, 4) for k = 2 (ordering 11, 12, 22) and (1, 2, 4, 8) for k = 3."""
    u = np.array([[1.0], [2.0]])
    assert np.array_equal(opinf.khatri_rao_pow(u, 2).ravel(), [1.0, 2.0, 4.0])
    assert np.array_equal(opinf.khatri_rao_pow(u, 3).ravel(), [1.0, 2.0, 4.0, 8.0])
    assert opinf.khatri_rao_pow(np.ones((5, 3)), 3).shape == (35, 3) == (opinf.n_poly(5, 3), 3)


def test_compressed_power_equals_symmetric_kronecker():
    """A symmetric operator on the full Kronecker power equals its compressed parameterisation on the
    compressed power: H (u kron u) = Hc u*2, with Hc[:, ij] = H[:, ij] + H[:, ji] (i < j), H[:, ii]."""
    rng = np.random.default_rng(4)
    r = 5
    u = rng.standard_normal(r)
    H = rng.standard_normal((3, r * r))
    Hc = []
    for i in range(r):
        for j in range(i, r):
            Hc.append(H[:, i * r + j] + (H[:, j * r + i] if j != i else 0.0))
    Hc = np.array(Hc).T
    assert np.allclose(H @ np.kron(u, u), Hc @ opinf.khatri_rao_pow(u[:, None], 2).ravel(), rtol=1e-13, atol=1e-13)
    C = rng.standard_normal((3, r ** 3))
    Cc = np.zeros((3, opinf.n_poly(r, 3)))
    col = 0
    for i in range(r):
        for j in range(i, r):
            for l in range(j, r):
                for a, b, c in set(itertools.permutations((i, j, l))):
                    Cc[:, col] += C[:, a * r * r + b * r + c]
                col += 1
    assert np.allclose(C @ np.kron(np.kron(u, u), u), Cc @ opinf.khatri_rao_pow(u[:, None], 3).ravel(),
                       rtol=1e-12, atol=1e-12)


def _poly_system(rng, r=4, rb=2, order=3, scale=0.3):
    K = rng.standard_normal((r, r))
    B = rng.standard_normal((r, rb))
    H = scale * rng.standard_normal((r, opinf.n_poly(r, 2))) if order >= 2 else None
    C = scale * rng.standard_normal((r, opinf.n_poly(r, 3))) if order >= 3 else None
    return K, B, H, C


def _accel(U, G, K, B, H, C):
    Y = -K @ U + B @ G
    if H is not None:
        Y -= H @ opinf.khatri_rao_pow(U, 2)
    if C is not None:
        Y -= C @ opinf.khatri_rao_pow(U, 3)
    return Y


@pytest.mark.parametrize("order", [1, 2, 3])
def test_opinf_recovers_known_polynomial_operators(order):
    """data generated exactly by a known reduced polynomial ODE, exact accelerations, lambda = 0,
    full column rank -> the fit recovers Kbar, Hbar, Cbar, Bbar (P:L278-285 consistency)."""
    rng = np.random.default_rng(10 + order)
    K, B, H, C = _poly_system(rng, order=order)
    U = rng.standard_normal((4, 400))
    G = rng.standard_normal((2, 400))
    Kf, Bf, Hf, Cf = opinf.opinf_fit_accel(U, G, _accel(U, G, K, B, H, C), 0.0, order)
    assert np.abs(Kf - K).max() < 1e-9 and np.abs(Bf - B).max() < 1e-9
    if order >= 2:
        assert np.abs(Hf - H).max() < 1e-9
    if order >= 3:
        assert np.abs(Cf - C).max() < 1e-9


def test_opinf_superset_model_and_ridge_limit():
    """quadratic data fitted with the cubic model -> Cbar ~ 0; lambda -> infinity -> 0."""
    rng = np.random.default_rng(21)
    K, B, H, _ = _poly_system(rng, order=2)
    U = rng.standard_normal((4, 400))
    G = rng.standard_normal((2, 400))
    Y = _accel(U, G, K, B, H, None)
    Kf, Bf, Hf, Cf = opinf.opinf_fit_accel(U, G, Y, 0.0, 3)
    assert np.linalg.norm(Cf) < 1e-8 * np.linalg.norm(Kf)
    Kl, Bl, Hl, Cl = opinf.opinf_fit_accel(U, G, Y, 1e12, 3)
    assert max(np.abs(x).max() for x in (Kl, Bl, Hl, Cl)) < 1e-6


def test_rom_accel_with_polynomial_terms_matches_kronecker_form():
    """oracle ROM.accel with Hbar, Cbar = e (-Kbar u - H_full (u kron u) - C_full (u kron u kron u) + Bbar g)
    with the full symmetric tensors rebuilt from the compressed ones (independent evaluation)."""
    from oracle import schwarz
    cfg = I.config("c2")
    boxes = [fem.Box(s["lo"], s["hi"], s["nel"]) for s in cfg["subdomains"]]
    faces = schwarz.detect_schwarz_faces(boxes)
    sub = cfg["subdomains"][1]
    codes = fem.dof_codes(boxes[1], sub["dirichlet"], faces[1].keys()).reshape(-1)
    nf, ns = int((codes == fem.FREE).sum()), int((codes == fem.SCHWARZ).sum())
    r, rb = 4, 3
    rng = np.random.default_rng(5)
    K, B, H, C = _poly_system(rng, r=r, rb=rb, order=3)
    ops = dict(Phi=np.linalg.qr(rng.standard_normal((nf, r)))[0], Phi_s=np.linalg.qr(rng.standard_normal((ns, rb)))[0],
               Kbar=K, Bbar=B, Hbar=H, Cbar=C)
    m = schwarz.ROM(sub, faces[1], cfg["E"], cfg["nu"], cfg["rho"], cfg["dt"], ops, e_scale=np.array([0.8, 1.1]))
    uh = rng.standard_normal((2, r))
    s = rng.standard_normal((2, ns))
    got = m.accel(uh, s)
    # full symmetric tensors: Hf[:, i r + j] = Hc[:, (i,j)] / multiplicity
    idx2 = [(i, j) for i in range(r) for j in range(i, r)]
    idx3 = [(i, j, l) for i in range(r) for j in range(i, r) for l in range(j, r)]
    Hf = np.zeros((r, r * r))
    for q, (i, j) in enumerate(idx2):
        perms = set(itertools.permutations((i, j)))
        for a, b in perms:
            Hf[:, a * r + b] = H[:, q] / len(perms)
    Cf = np.zeros((r, r ** 3))
    for q, (i, j, l) in enumerate(idx3):
        perms = set(itertools.permutations((i, j, l)))
        for a, b, c in perms:
            Cf[:, a * r * r + b * r + c] = C[:, q] / len(perms)
    for bidx, e in enumerate((0.8, 1.1)):
        u = uh[bidx]
        g = ops["Phi_s"].T @ s[bidx]
        ref = e * (-K @ u - Hf @ np.kron(u, u) - Cf @ np.kron(np.kron(u, u), u) + B @ g)
        assert np.allclose(got[bidx], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
