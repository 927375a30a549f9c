"""Oracle: hex8 linear-elastic FE on a structured box, lumped mass, explicit Newmark.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Plain fp64 NumPy, written as the
definitions read, with no stencil precomputation:

  * material  sigma = lambda tr(eps) I + 2 mu eps,  eps = sym grad u           (A.1)
  * element   K_e[a,c,b,d] = sum_q w_q detJ sum_{j,l} dN_a/dX_j C_cjdl dN_b/dX_l
              with 2x2x2 Gauss points (+-1/sqrt3, w=1)                         (P:L129-137 eq:weak_form)
  * force     f = sum_e scatter(K_e u_e)   -- an element loop                  (P:L133-137 eq:matrix_vector_form)
  * mass      row-sum lumping of the consistent mass rho int N_a N_b          (P:L178 footnote, L783)
  * Dirichlet split into free / constrained DOFs
  * nonlinear materials (readings R35, R36): internal force of the weak form
        f_a = sum_e sum_q w_q detJ P(F_q) dN_a/dX(q),  F = I + grad u  (same element loop, 2x2x2 Gauss)
    with P = F S and  Saint Venant-Kirchhoff  S = lambda tr(E) I + 2 mu E, E = 1/2 (F^T F - I)  (A.2)
                      Neohookean  S = kappa/2 (det C - 1) C^-1 + mu (det C)^(-1/3) (I - tr(C)/3 C^-1),
                                  C = F^T F, kappa = lambda + 2 mu/3                              (A.3)
  * explicit Newmark beta=0, gamma=1/2 in predictor form (reading R1):
        u* = u + dt v + dt^2/2 a ; a' = -f(u*)/m ; v' = v + dt/2 (a + a')

Node id p = i + (nx+1)(j + (ny+1)k); arrays are node-major (n_nodes, 3).
Faces: 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+.
"""
from __future__ import annotations

import itertools

import numpy as np

FREE, DIRICHLET, SCHWARZ = 0, 1, 2

# Local node order (xi, eta, zeta) in {-1,+1}^3:  (---, +--, ++-, -+-, --+, +-+, +++, -++)
LOCAL_NODES = np.array([(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1),
                        (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)], dtype=np.float64)
GAUSS_1D = np.array([-1.0, 1.0]) / np.sqrt(3.0)


def lame(E, nu):
    """Lame constants: lambda = E nu/((1+nu)(1-2nu)), mu = E/(2(1+nu))."""
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


def elasticity_tensor(lam, mu):
    """Isotropic C_ijkl = lambda d_ij d_kl + mu (d_ik d_jl + d_il d_jk), so that sigma = C:eps (A.1)."""
    d = np.eye(3)
    return (lam * np.einsum("ij,kl->ijkl", d, d)
            + mu * (np.einsum("ik,jl->ijkl", d, d) + np.einsum("il,jk->ijkl", d, d)))


def p_wave_speed(E, nu, rho):
    lam, mu = lame(E, nu)
    return np.sqrt((lam + 2 * mu) / rho)


def shape_functions(xi):
    """Trilinear N_a(xi) = prod_d (1 + xi_d s_ad)/2 and dN_a/dxi_d."""
    xi = np.asarray(xi, dtype=np.float64)
    f = 0.5 * (1.0 + LOCAL_NODES * xi[None, :])  # (8,3): per-axis factors
    N = f.prod(axis=1)
    dN = np.empty((8, 3))
    for d in range(3):
        others = [e for e in range(3) if e != d]
        dN[:, d] = 0.5 * LOCAL_NODES[:, d] * f[:, others[0]] * f[:, others[1]]
    return N, dN


def gauss_points():
    return [np.array(p) for p in itertools.product(GAUSS_1D, GAUSS_1D, GAUSS_1D)]


def hex8_stiffness(h, E, nu):
    """K_e as (8,3,8,3) for a rectangular hex with edge lengths h (A.1)."""
    lam, mu = lame(E, nu)
    C = elasticity_tensor(lam, mu)
    h = np.asarray(h, dtype=np.float64)
    detJ = np.prod(h) / 8.0
    Ke = np.zeros((8, 3, 8, 3))
    for q in gauss_points():
        _, dNdxi = shape_functions(q)
        dNdX = dNdxi / (h[None, :] / 2.0)         # J = diag(h/2)
        Ke += detJ * np.einsum("aj,cjdl,bl->acbd", dNdX, C, dNdX)
    return Ke


def hex8_lumped_mass(h, rho):
    """Row-sum of the consistent element mass rho sum_q N_a N_b detJ (P:L178 footnote)."""
    detJ = np.prod(np.asarray(h, dtype=np.float64)) / 8.0
    Me = np.zeros((8, 8))
    for q in gauss_points():
        N, _ = shape_functions(q)
        Me += rho * detJ * np.outer(N, N)
    return Me.sum(axis=1)


class Box:
    """Structured hex8 mesh of the box [lo, hi] with nel elements per axis."""

    def __init__(self, lo, hi, nel):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.nel = tuple(int(n) for n in nel)
        if any(n < 1 for n in self.nel) or np.any(self.hi <= self.lo):
            raise ValueError("invalid box")
        self.h = (self.hi - self.lo) / np.asarray(self.nel, dtype=np.float64)
        self.nn = tuple(n + 1 for n in self.nel)
        self.n_nodes = self.nn[0] * self.nn[1] * self.nn[2]
        self.n_elems = self.nel[0] * self.nel[1] * self.nel[2]

    def node_id(self, i, j, k):
        return i + self.nn[0] * (j + self.nn[1] * k)

    def ijk(self, p):
        p = np.asarray(p)
        return p % self.nn[0], (p // self.nn[0]) % self.nn[1], p // (self.nn[0] * self.nn[1])

    def coords(self, nodes=None):
        if nodes is None:
            nodes = np.arange(self.n_nodes)
        i, j, k = self.ijk(nodes)
        return np.stack([self.lo[0] + i * self.h[0], self.lo[1] + j * self.h[1],
                         self.lo[2] + k * self.h[2]], axis=-1)

    def face_nodes(self, face):
        """Node ids on a closed face, ascending."""
        axis, side = face // 2, face % 2
        i, j, k = self.ijk(np.arange(self.n_nodes))
        idx = (i, j, k)[axis]
        return np.nonzero(idx == (self.nel[axis] if side else 0))[0]

    # element-loop helpers -------------------------------------------------
    def _grid(self, a):
        return a.reshape(self.nn[2], self.nn[1], self.nn[0], *a.shape[1:])

    def _slice(self, a_local):
        di, dj, dk = ((LOCAL_NODES[a_local] + 1) // 2).astype(int)
        nx, ny, nz = self.nel
        return (slice(dk, dk + nz), slice(dj, dj + ny), slice(di, di + nx))


def internal_force(box: Box, Ke: np.ndarray, u: np.ndarray) -> np.ndarray:
    """f = sum_e scatter(K_e u_e) over every element of the box (element loop)."""
    ug = box._grid(u)
    ue = np.stack([ug[box._slice(b)] for b in range(8)], axis=-2)   # (nz,ny,nx,8,3)
    ue = ue.reshape(-1, 24)
    fe = ue @ Ke.reshape(24, 24).T                                    # (nel, 24)
    fe = fe.reshape(box.nel[2], box.nel[1], box.nel[0], 8, 3)
    f = np.zeros_like(ug)
    for a in range(8):
        f[box._slice(a)] += fe[..., a, :]
    return f.reshape(-1, 3)


def internal_force_at(box: Box, Ke: np.ndarray, value_at, nodes) -> np.ndarray:
    """f at selected nodes only, summing K_e rows of the (up to 8) incident elements.
    value_at(node_ids) -> (len, 3) returns the displacement of arbitrary nodes."""
    nodes = np.asarray(nodes)
    out = np.zeros((len(nodes), 3))
    I, J, K = box.ijk(nodes)
    for n, (i, j, k) in enumerate(zip(I, J, K)):
        for a in range(8):
            # element whose local node a is (i,j,k)
            di, dj, dk = ((LOCAL_NODES[a] + 1) // 2).astype(int)
            ei, ej, ek = i - di, j - dj, k - dk
            if not (0 <= ei < box.nel[0] and 0 <= ej < box.nel[1] and 0 <= ek < box.nel[2]):
                continue
            enodes = [box.node_id(ei + int((LOCAL_NODES[b][0] + 1) // 2), ej + int((LOCAL_NODES[b][1] + 1) // 2),
                                  ek + int((LOCAL_NODES[b][2] + 1) // 2)) for b in range(8)]
            ue = value_at(np.array(enodes))                            # (8,3)
            out[n] += np.einsum("cbd,bd->c", Ke[a], ue)
    return out


def lumped_mass(box: Box, rho: float) -> np.ndarray:
    me = hex8_lumped_mass(box.h, rho)
    m = np.zeros((box.nn[2], box.nn[1], box.nn[0]))
    for a in range(8):
        m[box._slice(a)] += me[a]
    return m.reshape(-1)


def assembled_stiffness(box: Box, Ke: np.ndarray) -> np.ndarray:
    """Brute-force dense K (3n x 3n, DOF id 3p+c) for tiny meshes (pin for the element loop)."""
    n = box.n_nodes
    K = np.zeros((3 * n, 3 * n))
    Ke24 = Ke.reshape(24, 24)
    for ek in range(box.nel[2]):
        for ej in range(box.nel[1]):
            for ei in range(box.nel[0]):
                en = [box.node_id(ei + int((LOCAL_NODES[b][0] + 1) // 2), ej + int((LOCAL_NODES[b][1] + 1) // 2),
                                  ek + int((LOCAL_NODES[b][2] + 1) // 2)) for b in range(8)]
                dofs = np.array([3 * p + c for p in en for c in range(3)])
                K[np.ix_(dofs, dofs)] += Ke24
    return K


def dof_codes(box: Box, dirichlet, schwarz_faces) -> np.ndarray:
    """Per-DOF constraint code (n_nodes,3): Dirichlet > Schwarz > free (reading R12, R13).
    dirichlet: 6 bitmasks (1:x,2:y,4:z); schwarz_faces: iterable of face ids."""
    codes = np.full((box.n_nodes, 3), FREE, dtype=np.int8)
    for f in schwarz_faces:
        codes[box.face_nodes(f), :] = SCHWARZ
    for f in range(6):
        for c in range(3):
            if dirichlet[f] >> c & 1:
                codes[box.face_nodes(f), c] = DIRICHLET
    return codes


def explicit_newmark_step(u, v, a, s_values, codes, schwarz_dofs, force, m, dt):
    """One explicit Newmark (beta=0, gamma=1/2) step in predictor form (c.1 step 7, reading R1).

    u, v, a: checkpoint state (n,3); s_values: prescribed values at the Schwarz DOFs,
    in the order of `schwarz_dofs` (flat DOF ids 3p+c); force(u*) -> (n,3); m: (n,) lumped mass.
    Returns (u*, v', a'); v', a' are zero on constrained DOFs (reading R10)."""
    free = codes == FREE
    ustar = np.where(free, u + dt * v + 0.5 * dt * dt * a, 0.0)
    ustar.reshape(-1)[schwarz_dofs] = s_values
    f = force(ustar)
    a_new = np.where(free, -f / m[:, None], 0.0)
    v_new = np.where(free, v + 0.5 * dt * (a + a_new), 0.0)
    return ustar, v_new, a_new


# ---------------------------------------------------------------------------------------
# nonlinear materials (App. A.2/A.3; readings R35, R36)
# ---------------------------------------------------------------------------------------

def pk1_svk(F, lam, mu):
    """Saint Venant-Kirchhoff: E = 1/2 (F^T F - I) (reading R35: the printed "1/2 F^T F - I" at P:L1961 is a
    typo, its own expansion at P:L1975 is 1/2 (F^T F - I)), S = lambda tr(E) I + 2 mu E (eq:svk_S),
    P = F S (eq:svk_P).  F: (..., 3, 3)."""
    I = np.eye(3)
    E = 0.5 * (np.swapaxes(F, -1, -2) @ F - I)
    trE = np.trace(E, axis1=-2, axis2=-1)
    S = lam * trE[..., None, None] * I + 2.0 * mu * E
    return F @ S


def pk1_neohookean(F, kappa, mu):
    """Neohookean (A.3): C = F^T F, S_vol = kappa/2 (det C - 1) C^-1,
    S_dev = mu (det C)^(-1/3) (I - tr(C)/3 C^-1) (reading R36: S = 2 dA/dC of A_dev = mu/2 ((det C)^(-1/3)
    tr C - 3), eq:Adev P:L2005; the printed 1/2 in front of C^-1 tr C at P:L2017 is inconsistent with it),
    P = F S."""
    I = np.eye(3)
    C = np.swapaxes(F, -1, -2) @ F
    detC = np.linalg.det(C)
    Ci = np.linalg.inv(C)
    trC = np.trace(C, axis1=-2, axis2=-1)
    S = (0.5 * kappa * (detC - 1.0))[..., None, None] * Ci \
        + (mu * detC ** (-1.0 / 3.0))[..., None, None] * (I - (trC / 3.0)[..., None, None] * Ci)
    return F @ S


def material_pk1(material, E, nu):
    """P(F) for material 'svk' | 'neohookean' with the Lame constants of (E, nu); kappa = lambda + 2 mu/3."""
    lam, mu = lame(E, nu)
    if material == "svk":
        return lambda F: pk1_svk(F, lam, mu)
    if material == "neohookean":
        return lambda F: pk1_neohookean(F, lam + 2.0 * mu / 3.0, mu)
    raise ValueError(material)


def internal_force_nonlinear(box: Box, u: np.ndarray, pk1) -> np.ndarray:
    """f_a = sum_e sum_q w_q detJ P(F_q) dN_a/dX(q), F_q = I + sum_b u_b (x) dN_b/dX(q)  (weak form
    P:L129-137 with the material's first Piola-Kirchhoff stress; element loop, 2x2x2 Gauss, w = 1)."""
    ug = box._grid(u)
    ue = np.stack([ug[box._slice(b)] for b in range(8)], axis=-2).reshape(-1, 8, 3)   # (nel, 8, 3)
    h = box.h
    detJ = np.prod(h) / 8.0
    fe = np.zeros_like(ue)
    for q in gauss_points():
        _, dNdxi = shape_functions(q)
        dNdX = dNdxi / (h[None, :] / 2.0)
        G = np.einsum("eai,aj->eij", ue, dNdX)        # (grad u)_ij = du_i/dX_j
        P = pk1(np.eye(3) + G)
        fe += detJ * np.einsum("eij,aj->eai", P, dNdX)
    fe = fe.reshape(box.nel[2], box.nel[1], box.nel[0], 8, 3)
    f = np.zeros_like(ug)
    for a in range(8):
        f[box._slice(a)] += fe[..., a, :]
    return f.reshape(-1, 3)
