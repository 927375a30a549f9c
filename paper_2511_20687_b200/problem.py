"""Set up a BASELINE workload (osam_inputs.config) on libosam.so: marshalling only.

Builds one `Subdomain` per box of the workload, uploads the seeded initial condition
(node-major arrays from osam_inputs are transposed to the ABI's SoA layout), runs
osam_step and reads states back.  No arithmetic of the method happens here.
"""
from __future__ import annotations

import numpy as np

import osam_inputs

from .osam import OSAM_FOM, OSAM_ROM, Subdomain, osam_step


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
            rom = dict(Phi=o["Phi"], Phi_s=o["Phi_s"], Kbar=o["Kbar"], Bbar=o["Bbar"])
        subs.append(Subdomain(kind, s["lo"], s["hi"], s["nel"], cfg["E"], cfg["nu"], cfg["rho"], s["dirichlet"],
                              stream=stream, rom=rom, e_scale=e_scale(cfg) if kind == OSAM_ROM else None))
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
