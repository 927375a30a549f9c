"""Oracle: offline stage -- POD, boundary POD, ridge OpInf, training runs (Algorithm 2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). The operators this module writes
are inputs shared by both online paths (the CUDA library reads them through the C-ABI).

  * POD: thin SVD U = Phi Sigma Psi^T, Phi_r = first r columns (eq:pod_cutoff);
    Euclidean, uncentred; column signs fixed so the largest-|entry| is positive (R17).
  * Energy rule E_r = sum_{i<=r} s_i^2 / sum_i s_i^2 (P:L788-792 eq:pod_energy); the smallest r
    with E_r >= delta_E = 0.999999 (reading R16).
  * OpInf (P:L263-272 eq:quadratic_opinf; L609-614 eq:opinf_schwarz_inference):
        argmin_O || O [U^; G^; U^*2; U^*3] - D_t^2(U^) ||_F^2 + lambda ||O||_F^2 ,
        O = [-Kbar, Bbar, -Hbar, -Cbar]   (linear: order 1; QOpInf: order 2; COpInf: order 3)
    where U^*k is the compressed column-wise Khatri-Rao power (P:L167 footnote; S:L437-445:
    monomials u_i u_j, i <= j, and u_i u_j u_l, i <= j <= l, in lexicographic order)
    with U^ = Phi^T U, G^ = Phi_dS^T S and D_t^2 the central second difference on interior
    columns (reading R18), one lambda in SI units (R20), solved as augmented least squares.
  * Training recipes per reading R25.
  * Regularisation selection (grid P:L808; reading R34): for every lambda of the
    grid 1e-4 * 10^(4 (j-1)/(n-1)), j = 1..n (n = 40), fit the operators, replay the ROM alone
    with explicit Newmark and the Schwarz boundary data of the training run (g^_k = G^[:, k]),
    and score ||U^bar - U^hat||_F / ||U^bar||_F in reduced coordinates; lambda* = first argmin
    (non-finite errors never win).
"""
from __future__ import annotations

import numpy as np

from . import fem, schwarz


def pod(U, r):
    """First r left singular vectors (sign-fixed) and all singular values of U."""
    Phi, sigma, _ = np.linalg.svd(U, full_matrices=False)
    Phi = Phi[:, :r].copy()
    idx = np.argmax(np.abs(Phi), axis=0)
    sgn = np.sign(Phi[idx, np.arange(Phi.shape[1])])
    sgn[sgn == 0] = 1.0
    return Phi * sgn[None, :], sigma


def energy(sigma):
    """E_r for r = 1..len(sigma) (eq:pod_energy)."""
    s2 = np.asarray(sigma, dtype=np.float64) ** 2
    return np.cumsum(s2) / s2.sum()


def energy_rank(sigma, delta=0.999999):
    """Smallest r with E_r >= delta (reading R16)."""
    E = energy(sigma)
    return int(np.searchsorted(E, delta, side="left") + 1)


def second_difference(Ubar, dt):
    """D_t^2 on interior columns k = 1..K-2: (U_{k+1} - 2 U_k + U_{k-1}) / dt^2."""
    return (Ubar[:, 2:] - 2.0 * Ubar[:, 1:-1] + Ubar[:, :-2]) / (dt * dt)


def khatri_rao_pow(U, k):
    """Compressed column-wise Kronecker power of U (r x tau): rows u_i u_j (i <= j) for k = 2 and
    u_i u_j u_l (i <= j <= l) for k = 3, lexicographic; k = 1 returns U."""
    U = np.atleast_2d(np.asarray(U, dtype=np.float64))
    r = U.shape[0]
    if k == 1:
        return U
    rows = []
    if k == 2:
        for i in range(r):
            for j in range(i, r):
                rows.append(U[i] * U[j])
    elif k == 3:
        for i in range(r):
            for j in range(i, r):
                for l in range(j, r):
                    rows.append(U[i] * U[j] * U[l])
    else:
        raise ValueError("k in {1, 2, 3}")
    return np.array(rows)


def n_poly(r, k):
    """Length of the compressed k-th power: r (r+1) ... (r+k-1) / k!."""
    return {1: r, 2: r * (r + 1) // 2, 3: r * (r + 1) * (r + 2) // 6}[k]


def opinf_fit_accel(Ubar, Ghat, Ydd, lam, order=1):
    """Ridge OpInf with given reduced accelerations Ydd (columns = samples):
    argmin || Ydd + Kbar U + Hbar U*2 + Cbar U*3 - Bbar G ||_F^2 + lam ||[Kbar Hbar Cbar Bbar]||_F^2,
    solved as augmented least squares.  Returns (Kbar, Bbar, Hbar, Cbar); Hbar/Cbar are None
    below their order."""
    blocks = [Ubar, Ghat] + [khatri_rao_pow(Ubar, k) for k in range(2, order + 1)]
    D = np.vstack(blocks)
    n = D.shape[0]
    A = np.vstack([D.T, np.sqrt(lam) * np.eye(n)])
    b = np.vstack([Ydd.T, np.zeros((n, Ydd.shape[0]))])
    Ot, *_ = np.linalg.lstsq(A, b, rcond=None)
    O = Ot.T                                             # (r, n)
    r, rb = Ubar.shape[0], Ghat.shape[0]
    Kbar, Bbar = -O[:, :r], O[:, r:r + rb]
    Hbar = -O[:, r + rb:r + rb + n_poly(r, 2)] if order >= 2 else None
    Cbar = -O[:, r + rb + n_poly(r, 2):] if order >= 3 else None
    return Kbar, Bbar, Hbar, Cbar


def opinf_fit(Ubar, Ghat, dt, lam, order=1):
    """Ridge OpInf for  u^'' + Kbar u^ (+ Hbar u^*2 + Cbar u^*3) = Bbar g^  from projected snapshots
    (columns = time), accelerations by central differences on the interior columns (reading R18).
    order 1 returns (Kbar, Bbar); orders 2, 3 return (Kbar, Bbar, Hbar, Cbar)."""
    Y = second_difference(Ubar, dt)                      # (r, K-2)
    out = opinf_fit_accel(Ubar[:, 1:-1], Ghat[:, 1:-1], Y, lam, order)
    return out[:2] if order == 1 else out


def build_rom_operators(U, S, dt, r, lam, delta=0.999999, r_b=None, order=1):
    """Phi, Phi_dS, Kbar, Bbar (and Hbar, Cbar for order 2, 3) from snapshot matrices U (n_free x K)
    and S (n_s x K)."""
    Phi, sigma = pod(U, r)
    Phi_s_full, sigma_s = pod(S, min(S.shape))
    if r_b is None:
        r_b = energy_rank(sigma_s, delta)
    Phi_s = Phi_s_full[:, :r_b]
    Kbar, Bbar, Hbar, Cbar = opinf_fit_accel(*_fit_data(Phi.T @ U, Phi_s.T @ S, dt), lam, order)
    ops = dict(Phi=Phi, Phi_s=Phi_s, Kbar=Kbar, Bbar=Bbar, sigma=sigma, sigma_s=sigma_s,
               r=r, r_b=r_b, lam=lam, dt=dt, order=order)
    if order >= 2:
        ops["Hbar"] = Hbar
    if order >= 3:
        ops["Cbar"] = Cbar
    return ops


def _fit_data(Ubar, Ghat, dt):
    return Ubar[:, 1:-1], Ghat[:, 1:-1], second_difference(Ubar, dt)


# ---------------------------------------------------------------------------------------
# training runs (reading R25)
# ---------------------------------------------------------------------------------------

def _online_models_codes(cfg):
    boxes = [fem.Box(s["lo"], s["hi"], s["nel"]) for s in cfg["subdomains"]]
    faces = schwarz.detect_schwarz_faces(boxes)
    return boxes, faces


def training_snapshots_single_domain(cfg, inputs):
    """c2: single-domain FOM on the training box, snapshots at steps 0..n-1 restricted to each ROM
    sub-block (nodes with x >= lo of the ROM box; conformal).  Returns {i: (X_free, X_schwarz)}."""
    tr = cfg["rom"]["training"]
    dom = tr["domain"]
    train_cfg = dict(cfg, subdomains=[dom])
    m = schwarz.build_models(train_cfg)[0]
    u0 = inputs.initial_displacements(cfg, dom)
    state = m.init_state(u0)
    snaps = [state["u"][0].copy()]
    for _ in range(tr["n_snapshots"] - 1):
        state = m.advance(state, np.zeros((1, 0)))
        snaps.append(state["u"][0].copy())
    boxes, faces = _online_models_codes(cfg)
    out = {}
    for i, s in enumerate(cfg["subdomains"]):
        if s["kind"] != "rom":
            continue
        rb = boxes[i]
        tb = m.box
        off = np.rint((rb.lo - tb.lo) / tb.h).astype(int)
        assert np.allclose(rb.h, tb.h), "c2 training restriction assumes a conformal sub-block"
        I, J, K = rb.ijk(np.arange(rb.n_nodes))
        tnodes = tb.node_id(I + off[0], J + off[1], K + off[2])
        codes = fem.dof_codes(rb, s["dirichlet"], faces[i].keys()).reshape(-1)
        free = np.nonzero(codes == fem.FREE)[0]
        sd = np.nonzero(codes == fem.SCHWARZ)[0]
        X = np.stack([u[tnodes].reshape(-1) for u in snaps], axis=1)      # (3 n_rom, K)
        out[i] = (X[free], X[sd])
    return out


def train_single_domain(cfg, inputs):
    """c2: operators from the single-domain training snapshots."""
    return {i: build_rom_operators(Xf, Xs, cfg["dt"], cfg["rom"]["r"], cfg["rom"]["lam"], cfg["rom"]["energy"],
                                   order=cfg["rom"].get("order", 1))
            for i, (Xf, Xs) in training_snapshots_single_domain(cfg, inputs).items()}


def train_coupled(cfg, inputs):
    """c4/c5: FOM-FOM(-FOM) O-SAM on the training meshes, all snapshots 0..n_steps (top-down
    training, Algorithm 2 steps 1-2)."""
    tr = cfg["rom"]["training"]
    train_cfg = dict(cfg, subdomains=tr["subdomains"], batch=1)
    models = schwarz.build_models(train_cfg)
    u0s = [inputs.initial_displacement(train_cfg, s)[None] for s in tr["subdomains"]]
    snaps = [[] for _ in models]

    rom_ids = [i for i, s in enumerate(cfg["subdomains"]) if s["kind"] == "rom"]

    def record(states):   # only the subdomains that become ROMs online (storage; c4: 1.6M DOFs x 501 each)
        for i in rom_ids:
            snaps[i].append(states[i]["u"][0].reshape(-1).copy())

    states = [m.init_state(u0) for m, u0 in zip(models, u0s)]
    record(states)
    for _ in range(tr["n_steps"]):
        states, _ = schwarz.controller_step(models, states, cfg["tol"], cfg["max_iters"], cfg["min_iters"])
        record(states)
    ops = {}
    for i, s in enumerate(cfg["subdomains"]):
        if s["kind"] != "rom":
            continue
        m = models[i]
        X = np.stack(snaps[i], axis=1)
        snaps[i] = None
        ops[i] = build_rom_operators(X[m.free_dofs], X[m.schwarz_dofs], cfg["dt"], cfg["rom"]["r"],
                                     cfg["rom"]["lam"], cfg["rom"]["energy"], order=cfg["rom"].get("order", 1))
    return ops


def train(cfg, inputs):
    kind = cfg["rom"]["training"]["kind"]
    if kind == "single_domain":
        return train_single_domain(cfg, inputs)
    return train_coupled(cfg, inputs)


# ---------------------------------------------------------------------------------------
# regularisation selection by subdomain-local replay (reading R34)
# ---------------------------------------------------------------------------------------

def lambda_grid(n=40):
    """lambda_j = 1e-4 * 10^(4 (j-1)/(n-1)), j = 1..n."""
    return 1e-4 * 10.0 ** (4.0 / (n - 1) * np.arange(n))


def replay_accel(O, order, r, r_b, u, g):
    """a^ = O [u; g; u^*2; u^*3] with O = [-Kbar, Bbar, -Hbar, -Cbar] (r x (r + r_b + nf))."""
    z = [u, g]
    if order >= 2:
        z.append(khatri_rao_pow(u[:, None], 2)[:, 0])
    if order >= 3:
        z.append(khatri_rao_pow(u[:, None], 3)[:, 0])
    return O @ np.concatenate(z)


def rom_replay(O, Ubar, Ghat, dt, order=1, vh0=None):
    """Subdomain-local replay: the OpInf ROM alone, explicit Newmark (c.1 step 10 form),
    from u^_0 = Ubar[:, 0], v^_0 = vh0 (0: the training runs start at rest), with the Schwarz boundary
    data of the training run, g^_k = Ghat[:, k].  Returns U^hat (r x K)."""
    r, K = Ubar.shape
    r_b = Ghat.shape[0]
    u = Ubar[:, 0].copy()
    v = np.zeros(r) if vh0 is None else np.asarray(vh0, dtype=np.float64).copy()
    a = replay_accel(O, order, r, r_b, u, Ghat[:, 0])
    out = np.empty((r, K))
    out[:, 0] = u
    with np.errstate(all="ignore"):
        for k in range(1, K):
            u = u + dt * v + 0.5 * dt * dt * a
            an = replay_accel(O, order, r, r_b, u, Ghat[:, k])
            v = v + 0.5 * dt * (a + an)
            a = an
            out[:, k] = u
    return out


def trajectory_error(Ubar, Uhat):
    """||Ubar - Uhat||_F / ||Ubar||_F (reduced coordinates; reading R34)."""
    with np.errstate(all="ignore"):
        return float(np.sqrt(np.sum((Ubar - Uhat) ** 2)) / np.sqrt(np.sum(Ubar ** 2)))


def operator_matrix(ops, order=1):
    """O = [-Kbar, Bbar, -Hbar, -Cbar] of a fit."""
    Kbar, Bbar = ops[0], ops[1]
    blocks = [-Kbar, Bbar]
    if order >= 2:
        blocks.append(-ops[2])
    if order >= 3:
        blocks.append(-ops[3])
    return np.concatenate(blocks, axis=1)


def select_lambda(Ubar, Ghat, dt, grid=None, order=1):
    """lambda* of the grid by subdomain-local replay.  Returns (index, errors (n,), operator matrices)."""
    grid = lambda_grid() if grid is None else np.asarray(grid)
    errs, Os = [], []
    for lam in grid:
        O = operator_matrix(opinf_fit(Ubar, Ghat, dt, lam, order), order)
        Os.append(O)
        errs.append(trajectory_error(Ubar, rom_replay(O, Ubar, Ghat, dt, order)))
    errs = np.array(errs)
    score = np.where(np.isfinite(errs), errs, np.inf)
    return int(np.argmin(score)), errs, Os
