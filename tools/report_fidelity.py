"""Report-only outputs of SURVEY 8(c) c.1 step 13 for the trained-ROM configurations (calls only oracle/):

  * the ROM growth factor  max_k ||u^(t_k)|| / ||u^(t_0)||  per ROM subdomain (and sample);
  * fidelity by eq:mse:  E_Omega(u) = sqrt(sum_k ||u(t_k) - u_ref(t_k)||^2) / sqrt(sum_k ||u_ref(t_k)||^2)
    with u_ref the FOM solution of the subdomain in a FOM-FOM O-SAM run on the same meshes (the paper's reference,
    P:L799-800); a ROM subdomain's field is Phi u^ on its free DOFs and its Schwarz values (the oracle's
    full_field), compared over all DOFs.

    python tools/report_fidelity.py [c2] [c5] [--c5-samples 4] > profiles/r3_fidelity.json

c2 runs its full 1000 steps; c5 its 2000 steps on the first `--c5-samples` samples of its seeded batch (each sample
needs its own FOM-FOM reference run).  A report, not a pin: the literal training settings give inaccurate or
unstable ROMs (SURVEY finding 7), which these numbers quantify.
"""
from __future__ import annotations

import argparse
import copy
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import osam_inputs as I  # noqa: E402
from oracle import opinf, schwarz  # noqa: E402


def fields(models, states):
    out = []
    for m, st in zip(models, states):
        out.append(st["u"].reshape(st["u"].shape[0], -1) if m.kind == "fom" else
                   m.full_field(st).reshape(st["uh"].shape[0], -1))
    return out


def run_pair(cfg, ops, e_scale, n_steps):
    """(per-step fields of the configured run, per-step fields of the FOM-FOM reference, growth factors)."""
    models = schwarz.build_models(cfg, rom_ops=ops, e_scale=e_scale)
    ref_cfg = copy.deepcopy(cfg)
    for s in ref_cfg["subdomains"]:
        s["kind"] = "fom"
    ref_cfg["batch"] = 1
    u0 = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    st = [m.init_state(u) for m, u in zip(models, u0)]
    rom_norm0 = [np.linalg.norm(s["uh"], axis=1) if m.kind == "rom" else None for m, s in zip(models, st)]
    growth = [np.ones_like(n) if n is not None else None for n in rom_norm0]
    acc = None
    refs = []
    B = max(m.batch for m in models)
    for b in range(B):
        rc = copy.deepcopy(ref_cfg)
        E = cfg["E"] * (e_scale[b] if e_scale is not None else 1.0)
        rc["E"] = E
        rm = schwarz.build_models(rc)
        rs = [m.init_state(u[b:b + 1]) for m, u in zip(rm, u0)]
        refs.append((rm, rs))
    num = np.zeros((len(models), B))
    den = np.zeros((len(models), B))

    def accumulate():
        f = fields(models, st)
        for b, (rm, rs) in enumerate(refs):
            fr = fields(rm, rs)
            for i in range(len(models)):
                num[i, b] += np.sum((f[i][b if f[i].shape[0] > 1 else 0] - fr[i][0]) ** 2)
                den[i, b] += np.sum(fr[i][0] ** 2)

    accumulate()
    for _ in range(n_steps):
        st, _ = schwarz.controller_step(models, st, cfg["tol"], cfg["max_iters"], cfg["min_iters"])
        for b, (rm, rs) in enumerate(refs):
            refs[b] = (rm, schwarz.controller_step(rm, rs, cfg["tol"], cfg["max_iters"], cfg["min_iters"])[0])
        for i, (m, s) in enumerate(zip(models, st)):
            if m.kind == "rom":
                with np.errstate(all="ignore"):
                    growth[i] = np.maximum(growth[i], np.linalg.norm(s["uh"], axis=1) / rom_norm0[i])
        accumulate()
    with np.errstate(all="ignore"):
        mse = np.sqrt(num) / np.sqrt(den)
    return mse, growth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c5"])
    ap.add_argument("--c5-samples", type=int, default=4)
    args = ap.parse_args()
    out = {"source": "tools/report_fidelity.py (oracle only)", "metric": "eq:mse P:L796-800 vs the FOM-FOM O-SAM "
           "reference on the same meshes; growth = max_k ||u^(t_k)|| / ||u^(t_0)||"}
    for name in args.configs:
        t0 = time.time()
        cfg = I.config(name)
        ops = opinf.train(cfg, I)
        e = None
        if name == "c5":
            nb = args.c5_samples
            cfg["samples"] = {k: tuple(v[:nb]) for k, v in cfg["samples"].items()}
            cfg["batch"] = nb
            e = np.asarray(cfg["samples"]["E"]) / cfg["E"]
        mse, growth = run_pair(cfg, ops, e, cfg["n_steps"])
        out[name] = {"steps": cfg["n_steps"], "samples": cfg.get("batch", 1),
                     "subdomains": [s["kind"] for s in cfg["subdomains"]],
                     "mse_per_subdomain_per_sample": mse.tolist(),
                     "rom_growth_per_subdomain_per_sample": [None if g is None else g.tolist() for g in growth],
                     "r": cfg["rom"]["r"], "r_b": {str(i): int(o["r_b"]) for i, o in ops.items()},
                     "seconds": round(time.time() - t0, 1)}
        print(json.dumps(out[name]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
