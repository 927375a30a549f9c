"""Set up a BASELINE workload (osam_inputs.config) on libosam.so: marshalling only.

Builds one `Subdomain` per box of the workload, uploads the seeded initial condition
(node-major arrays from osam_inputs are transposed to the ABI's SoA layout), runs
osam_step and reads states back.  No arithmetic of the method happens here.
"""
from __future__ import annotations

import numpy as np

import osam_inputs

from .osam import MATERIALS, OSAM_EXPLICIT, OSAM_FOM, OSAM_IMPLICIT, OSAM_LINEAR, OSAM_ROM, Subdomain, osam_step


def e_scale(cfg):
    if cfg.get("batch", 1) > 1:
        return np.asarray(cfg["samples"]["E"], dtype=np.float64) / cfg["E"]
    return None


def build(cfg, rom_ops=None, stream=None):
    subs = []
    for i, s in enumerate(cfg["subdomains"]):
        kind = OSAM_FOM if s["kind"] == "fom" else OSAM_ROM
        rom = None
        if kind == OSAM_ROM:
            o = rom_ops[i]
            rom = dict(Phi=o["Phi"], Phi_s=o["Phi_s"], Kbar=o["Kbar"], Bbar=o["Bbar"], Hbar=o.get("Hbar"),
                       Cbar=o.get("Cbar"), phi_rows=o.get("phi_rows"), n_free=o.get("n_free"))
        integ = OSAM_IMPLICIT if s.get("integrator", "explicit") == "implicit" else OSAM_EXPLICIT
        subs.append(Subdomain(kind, s["lo"], s["hi"], s["nel"], cfg["E"], cfg["nu"], cfg["rho"], s["dirichlet"],
                              stream=stream, rom=rom, e_scale=e_scale(cfg) if kind == OSAM_ROM else None,
                              n_substeps=s.get("n_sub", 1), integrator=integ,
                              material=MATERIALS[s.get("material", cfg.get("material", "linear"))]
                              if kind == OSAM_FOM else OSAM_LINEAR))
    return subs


def soa(u_nodes):
    """(batch, n, 3) node-major -> contiguous (batch, 3, n) SoA as the ABI expects."""
    return np.ascontiguousarray(np.asarray(u_nodes, dtype=np.float64).transpose(0, 2, 1))


def initial_fields(cfg):
    return [soa(osam_inputs.initial_displacements(cfg, s)) for s in cfg["subdomains"]]


def set_ics(cfg, subs, device=None, fields=None):
    """Upload the seeded IC; `device` (e.g. 'cuda:0') stages it in a torch tensor first."""
    fields = fields if fields is not None else initial_fields(cfg)
    for sub, u0 in zip(subs, fields):
        if device is not None:
            import torch
            sub.set_ic(torch.from_numpy(u0).to(device))
        else:
            sub.set_ic(u0)


def dof_split(cfg, i):
    """(n_free, n_s) of subdomain i: the Schwarz faces of a box are the faces strictly inside another
    box of the workload and laterally covered by it (include/osam.h conventions); Dirichlet components
    win.  Host-side bookkeeping used to size stand-in ROM operators before the library binds the group."""
    subs = cfg["subdomains"]
    a = subs[i]
    nn = [n + 1 for n in a["nel"]]
    size = max(a["hi"][d] - a["lo"][d] for d in range(3))
    tol = 1e-12 * size
    sw = [False] * 6
    for f in range(6):
        ax = f // 2
        x = a["hi"][ax] if f % 2 else a["lo"][ax]
        for j, b in enumerate(subs):
            if j == i:
                continue
            inside = b["lo"][ax] + tol < x < b["hi"][ax] - tol
            lateral = all(b["lo"][d] <= a["lo"][d] + tol and a["hi"][d] <= b["hi"][d] + tol for d in range(3) if d != ax)
            if inside and lateral:
                sw[f] = True
                break
    idx = np.indices((nn[2], nn[1], nn[0])).reshape(3, -1)[::-1]  # i, j, k per node (node id order)
    on = [idx[f // 2] == ((nn[f // 2] - 1) if f % 2 else 0) for f in range(6)]
    swn = np.zeros(idx.shape[1], dtype=bool)
    for f in range(6):
        if sw[f]:
            swn |= on[f]
    n_free = n_s = 0
    for c in range(3):
        dirc = np.zeros(idx.shape[1], dtype=bool)
        for f in range(6):
            if (a["dirichlet"][f] >> c) & 1:
                dirc |= on[f]
        n_s += int((swn & ~dirc).sum())
        n_free += int((~swn & ~dirc).sum())
    return n_free, n_s


def synthetic_rom_ops(cfg, r_b=40, seed=7):
    """Stand-in reduced operators of the trained sizes for every ROM subdomain (osam_inputs)."""
    ops = {}
    for i, s in enumerate(cfg["subdomains"]):
        if s["kind"] == "rom":
            n_free, n_s = dof_split(cfg, i)
            ops[i] = osam_inputs.synthetic_rom_operators(n_free, n_s, cfg["rom"]["r"], r_b, cfg["dt"], seed + i)
    return ops


def run(cfg, subs, n_steps=None, max_iters=None):
    return osam_step(subs, cfg["dt"], cfg["tol"], cfg["n_steps"] if n_steps is None else n_steps,
                     max_iters=max_iters or cfg["max_iters"], min_iters=cfg["min_iters"])


def fom_state(sub, accel=False):
    """(u, v[, a]) as node-major (n, 3) host arrays."""
    n = sub.n_nodes
    u = np.empty(3 * n)
    v = np.empty(3 * n)
    sub.get_state(u, v)
    out = [u.reshape(3, n).T.copy(), v.reshape(3, n).T.copy()]
    if accel:
        a = np.empty(3 * n)
        sub.get_accel(a)
        out.append(a.reshape(3, n).T.copy())
    return out


def rom_state(sub, accel=False):
    """(u^, v^[, a^]) as (batch, r) host arrays."""
    B, r = sub.batch, sub.r
    u = np.empty(B * r)
    v = np.empty(B * r)
    sub.get_state(u, v)
    out = [u.reshape(B, r), v.reshape(B, r)]
    if accel:
        a = np.empty(B * r)
        sub.get_accel(a)
        out.append(a.reshape(B, r))
    return out
