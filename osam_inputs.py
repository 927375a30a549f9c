"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NO arithmetic of the method (no element, transfer, time-step,
Schwarz or OpInf computation). It only states the five BASELINE.json workloads as
data, draws the seeded random numbers they need, and evaluates the initial
condition (IC) formulas at mesh nodes so that both paths start from the same bytes.

Readings used:
  * R4  dt = 0.5 * h_min / c_p with c_p = sqrt((lambda + 2 mu)/rho)  (P:L863 at nu=0).
        c5 evaluates c_p at the largest sampled modulus bound E = 1.2e9.
  * R13 roller = x-component held at 0; clamp = all components held at 0.
  * R14 c1/c2/c5: u_x = A exp(-((x-0.5)/0.05)^2) exactly as BASELINE prints it;
        c3/c4: u = A d exp(-|X-x_c|^2/(2 sigma^2)), sigma=0.05, A=1e-3, d seeded unit.
  * R23 c4 geometry [0,1.1] / [1,2] / [1.9,3] x [0,1]^2.
  * R25 training data recipes (c2 single-domain 100x10x10, c4 FOM^3 on 80^3, c5 FOM-FOM).

Faces are numbered 0:x-, 1:x+, 2:y-, 3:y+, 4:z-, 5:z+.  A Dirichlet face entry is
a bitmask of held components (1:x, 2:y, 4:z).  Node id p = i + (nx+1)(j + (ny+1)k);
arrays returned here are node-major (n_nodes, 3) float64.
"""
from __future__ import annotations

import copy
import math

import numpy as np

ROLLER_X = 1
CLAMP = 7

E0 = 1.0e9
NU = 0.25
RHO = 1000.0


def _cp(E, nu, rho):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return math.sqrt((lam + 2 * mu) / rho)


def _sub(name, kind, lo, hi, nel, dirichlet=(0, 0, 0, 0, 0, 0)):
    return dict(name=name, kind=kind, lo=tuple(float(x) for x in lo),
                hi=tuple(float(x) for x in hi), nel=tuple(int(n) for n in nel),
                dirichlet=tuple(int(m) for m in dirichlet))


def _dt(subs, E=E0):
    h_min = min((s["hi"][d] - s["lo"][d]) / s["nel"][d] for s in subs for d in range(3))
    return 0.5 * h_min / _cp(E, NU, RHO)


def seeded_direction(seed):
    """d = normalize(rng.standard_normal(3)) with default_rng(seed)."""
    rng = np.random.default_rng(seed)
    d = rng.standard_normal(3)
    return d / np.linalg.norm(d)


def c5_samples(batch=64, seed=5):
    """E = 1e9 (0.8 + 0.4 U) first, then A = 1e-3 (0.5 + U)."""
    rng = np.random.default_rng(seed)
    E = 1e9 * (0.8 + 0.4 * rng.random(batch))
    A = 1e-3 * (0.5 + rng.random(batch))
    return E, A


def config(name: str) -> dict:
    """Return the workload description for c1..c5 (BASELINE.json configs[0..4])."""
    if name == "c1":
        subs = [_sub("omega1", "fom", (0, 0, 0), (0.6, 0.1, 0.1), (30, 5, 5), (ROLLER_X, 0, 0, 0, 0, 0)),
                _sub("omega2", "fom", (0.4, 0, 0), (1.0, 0.1, 0.1), (24, 4, 4), (0, ROLLER_X, 0, 0, 0, 0))]
        cfg = dict(subdomains=subs, n_steps=200, tol=1e-10,
                   ic=dict(kind="beam", A=1e-3))
    elif name == "c2":
        subs = [_sub("omega1", "fom", (0, 0, 0), (0.6, 0.1, 0.1), (60, 10, 10), (ROLLER_X, 0, 0, 0, 0, 0)),
                _sub("omega2", "rom", (0.4, 0, 0), (1.0, 0.1, 0.1), (60, 10, 10), (0, ROLLER_X, 0, 0, 0, 0))]
        cfg = dict(subdomains=subs, n_steps=1000, tol=1e-10,
                   ic=dict(kind="beam", A=1e-3),
                   rom=dict(r=20, lam=1e-8, energy=0.999999,
                            training=dict(kind="single_domain",
                                          domain=_sub("train", "fom", (0, 0, 0), (1.0, 0.1, 0.1), (100, 10, 10),
                                                      (ROLLER_X, ROLLER_X, 0, 0, 0, 0)),
                                          n_snapshots=400)))
    elif name == "c3":
        subs = [_sub("omega1", "fom", (0, 0, 0), (0.55, 1, 1), (141, 256, 256), (CLAMP, 0, 0, 0, 0, 0)),
                _sub("omega2", "fom", (0.45, 0, 0), (1, 1, 1), (110, 200, 200))]
        cfg = dict(subdomains=subs, n_steps=500, tol=1e-8,
                   ic=dict(kind="gauss3d", A=1e-3, sigma=0.05, center=(0.5, 0.5, 0.5),
                           direction=tuple(seeded_direction(3))))
    elif name == "c4":
        subs = [_sub("omegaL", "rom", (0, 0, 0), (1.1, 1, 1), (80, 80, 80), (CLAMP, 0, 0, 0, 0, 0)),
                _sub("omegaC", "fom", (1, 0, 0), (2, 1, 1), (256, 256, 256)),
                _sub("omegaR", "rom", (1.9, 0, 0), (3, 1, 1), (80, 80, 80))]
        train = [dict(s, kind="fom", nel=(80, 80, 80)) for s in subs]
        cfg = dict(subdomains=subs, n_steps=500, tol=1e-10,
                   ic=dict(kind="gauss3d", A=1e-3, sigma=0.05, center=(1.5, 0.5, 0.5),
                           direction=tuple(seeded_direction(4))),
                   rom=dict(r=200, lam=1e-8, energy=0.999999,
                            training=dict(kind="coupled", subdomains=train, n_steps=500)))
    elif name == "c5":
        subs = [_sub("omegaL", "rom", (0, 0, 0), (0.6, 0.1, 0.1), (60, 10, 10), (ROLLER_X, 0, 0, 0, 0, 0)),
                _sub("omegaR", "rom", (0.4, 0, 0), (1.0, 0.1, 0.1), (40, 8, 8), (0, ROLLER_X, 0, 0, 0, 0))]
        E, A = c5_samples()
        train = [dict(s, kind="fom") for s in subs]
        cfg = dict(subdomains=subs, n_steps=2000, tol=1e-10,
                   ic=dict(kind="beam", A=1e-3), batch=64,
                   samples=dict(E=tuple(E), A=tuple(A)),
                   rom=dict(r=400, lam=1e-8, energy=0.999999,
                            training=dict(kind="coupled", subdomains=train, n_steps=2000)))
    else:
        raise KeyError(name)
    cfg["name"] = name
    cfg.setdefault("batch", 1)
    cfg["E"], cfg["nu"], cfg["rho"] = E0, NU, RHO
    cfg["max_iters"] = 50
    cfg["min_iters"] = 2
    # R4: c5 uses the stiffest sample bound for a single dt shared by all samples.
    cfg["dt"] = _dt(cfg["subdomains"], E=1.2e9 if name == "c5" else E0)
    return cfg


def scaled(cfg: dict, factor: float, n_steps: int | None = None) -> dict:
    """A copy of cfg with every mesh coarsened by `factor` (nel -> max(1, round(nel/factor)));
    dt is re-derived from the new meshes. Used for oracle-sized parity cases."""
    out = copy.deepcopy(cfg)
    for s in out["subdomains"]:
        s["nel"] = tuple(max(1, int(round(n / factor))) for n in s["nel"])
    out["dt"] = _dt(out["subdomains"], E=1.2e9 if cfg["name"] == "c5" else E0)
    if n_steps is not None:
        out["n_steps"] = n_steps
    out["name"] = cfg["name"] + f"/x{factor:g}"
    return out


def node_coords(lo, hi, nel):
    """Node coordinates X_ijk = lo + (i h_x, j h_y, k h_z), node-major (n_nodes, 3)."""
    nx, ny, nz = nel
    h = [(hi[d] - lo[d]) / nel[d] for d in range(3)]
    i = np.arange(nx + 1)
    j = np.arange(ny + 1)
    k = np.arange(nz + 1)
    K, J, I = np.meshgrid(k, j, i, indexing="ij")
    X = np.stack([lo[0] + I * h[0], lo[1] + J * h[1], lo[2] + K * h[2]], axis=-1)
    return X.reshape(-1, 3)


def initial_displacement(cfg: dict, sub: dict, amplitude: float | None = None) -> np.ndarray:
    """Analytic IC evaluated at every node of `sub`'s mesh (R14). v0 = 0 everywhere."""
    X = node_coords(sub["lo"], sub["hi"], sub["nel"])
    ic = cfg["ic"]
    A = ic["A"] if amplitude is None else amplitude
    u = np.zeros_like(X)
    if ic["kind"] == "beam":
        u[:, 0] = A * np.exp(-((X[:, 0] - 0.5) / 0.05) ** 2)
    elif ic["kind"] == "gauss3d":
        c = np.asarray(ic["center"])
        r2 = ((X - c) ** 2).sum(axis=1)
        g = A * np.exp(-r2 / (2 * ic["sigma"] ** 2))
        u = g[:, None] * np.asarray(ic["direction"])[None, :]
    else:
        raise KeyError(ic["kind"])
    return u


def initial_displacements(cfg: dict, sub: dict) -> np.ndarray:
    """(batch, n_nodes, 3): per-sample IC (c5 scales the amplitude per sample)."""
    if cfg["batch"] == 1:
        return initial_displacement(cfg, sub)[None]
    return np.stack([initial_displacement(cfg, sub, a) for a in cfg["samples"]["A"]])


def random_state(n_nodes, seed, scale=1e-3):
    """Seeded random (u, v) fields for unit/parity tests of single operations."""
    rng = np.random.default_rng(seed)
    return scale * rng.standard_normal((n_nodes, 3)), scale * 1e3 * rng.standard_normal((n_nodes, 3))


def synthetic_rom_operators(n_free, n_s, r, r_b, dt, seed):
    """Seeded stand-in reduced operators of the trained sizes (timing of configurations whose offline
    stage is too large to run per benchmark, e.g. c4's 80^3 ROMs).  Not a trained
    ROM: Phi, Phi_s have random +-1/sqrt(rows) entries (nearly orthonormal columns), Kbar is diagonal
    with reduced frequencies below the explicit stability limit of dt, Bbar is small and random."""
    rng = np.random.default_rng(seed)
    Phi = np.asfortranarray((rng.integers(0, 2, size=(n_free, r), dtype=np.int8) * 2 - 1) / np.sqrt(n_free))
    Phi_s = np.asfortranarray((rng.integers(0, 2, size=(n_s, r_b), dtype=np.int8) * 2 - 1) / np.sqrt(n_s))
    omega = np.linspace(0.05, 0.5, r) / dt
    Kbar = np.asfortranarray(np.diag(omega ** 2))
    Bbar = np.asfortranarray(0.1 * rng.standard_normal((r, r_b)) / (dt * dt * np.sqrt(r_b)))
    return dict(Phi=Phi, Phi_s=Phi_s, Kbar=Kbar, Bbar=Bbar)
