"""Write full-size oracle golden data for the GPU long-horizon parity tests (calls only oracle/).

    python tools/gen_golden_fullsize.py c3 [--steps 500]
    python tools/gen_golden_fullsize.py c4 [--steps N]      (needs tools/gen_c4_rom.py's operators)

Runs the CPU oracle (oracle.schwarz.controller_step, Algorithm 1; the FOM force by the
C element loop oracle/cfem.c for these box sizes) on BASELINE's full-size configuration from the seeded
IC and records, into tests/golden/<cfg>_long.npz (+ a provenance .json):

  * the Schwarz iteration count of every controller step (eq:conv_criterion P:L443-467);
  * the convergence quantities (n, num, den) of every tested iteration of every step;
  * per subdomain and step: ||u|| (all DOFs), ||v||, ||a|| (free DOFs) for a FOM; u^, v^ for a ROM;
  * a seeded sample of FOM nodes (uniform, near the Schwarz faces, on the exterior faces, near the
    pulse) with u, v, a at the steps listed in RECORD.

No value here comes from the CUDA path.  The output is what tests/test_gpu_longhorizon.py compares the
library with, element by element.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import pickle
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import osam_inputs as I  # noqa: E402
from oracle import fem, schwarz  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_SAMPLE = 6000


def sample_nodes(model, rng, center):
    """Seeded FOM sample: 1/3 uniform, 1/4 within two node layers of a Schwarz face, 1/6 on exterior faces,
    the rest within 0.15 of the pulse centre; plus the 8 corners."""
    box = model.box
    n = box.n_nodes
    I_, J_, K_ = box.ijk(np.arange(n))
    idx = (I_, J_, K_)
    near_s = np.zeros(n, dtype=bool)
    for f in model.schwarz_faces:
        ax, side = f // 2, f % 2
        d = (box.nel[ax] - idx[ax]) if side else idx[ax]
        near_s |= d <= 2
    on_face = np.zeros(n, dtype=bool)
    for f in range(6):
        if f in model.schwarz_faces:
            continue
        ax, side = f // 2, f % 2
        on_face |= idx[ax] == (box.nel[ax] if side else 0)
    X = box.coords()
    near_c = np.linalg.norm(X - np.asarray(center)[None, :], axis=1) < 0.15
    picks = [rng.choice(n, N_SAMPLE // 3, replace=False),
             rng.choice(np.nonzero(near_s)[0], N_SAMPLE // 4, replace=False),
             rng.choice(np.nonzero(on_face)[0], N_SAMPLE // 6, replace=False)]
    nc = np.nonzero(near_c)[0]
    if len(nc):
        picks.append(rng.choice(nc, min(len(nc), N_SAMPLE - sum(len(p) for p in picks)), replace=False))
    picks.append(np.array([box.node_id(i, j, k) for i in (0, box.nel[0]) for j in (0, box.nel[1])
                           for k in (0, box.nel[2])]))
    return np.unique(np.concatenate(picks))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c3", "c4"])
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--record", type=str, default=None, help="comma-separated steps with node samples")
    ap.add_argument("--out", type=str, default=None)
    ap.add_argument("--resume", action="store_true", help="continue from var/<out>_ckpt.pkl")
    ap.add_argument("--stamp-ops", action="store_true",
                    help="c4: only (re)write rom_ops_id of var/c4_ops into the provenance .json")
    args = ap.parse_args()
    if args.stamp_ops:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import gen_c4_rom
        jp = os.path.join(GOLDEN, (args.out or "c4_long") + ".json")
        with open(jp) as fh:
            prov = json.load(fh)
        prov["rom_ops_id"] = gen_c4_rom.rom_ops_id(gen_c4_rom.load_full_ops())
        with open(jp, "w") as fh:
            json.dump(prov, fh, indent=1)
        print("rom_ops_id", prov["rom_ops_id"])
        return
    cfg = I.config(args.config)
    n_steps = args.steps or cfg["n_steps"]
    record = sorted({int(x) for x in args.record.split(",")}) if args.record else \
        sorted({s for s in (1, 10, 50, 100, 250, n_steps) if s <= n_steps})
    rom_ops = None
    if args.config == "c4":
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import gen_c4_rom
        rom_ops = gen_c4_rom.load_full_ops()
        args.rom_ops_id = gen_c4_rom.rom_ops_id(rom_ops)
    models = schwarz.build_models(cfg, rom_ops)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    states = [m.init_state(u0) for m, u0 in zip(models, u0s)]
    rng = np.random.default_rng(20251120)
    center = cfg["ic"]["center"]
    samples = {i: sample_nodes(m, rng, center) for i, m in enumerate(models) if m.kind == "fom"}
    iters = np.zeros(n_steps, dtype=np.int64)
    trace_n, trace_num, trace_den, trace_step = [], [], [], []
    norms = {i: [] for i in range(len(models))}
    vals = {i: [] for i in samples}
    ckpt_path = os.path.join(ROOT, "var", f"{args.out or args.config + '_long'}_ckpt.pkl")
    k0 = 1
    el0 = 0.0
    if args.resume and os.path.exists(ckpt_path):     # oracle state and records of an interrupted run
        with open(ckpt_path, "rb") as fh:
            ck = pickle.load(fh)
        states, iters[:len(ck["iters"])] = ck["states"], ck["iters"]
        trace_n, trace_num, trace_den, trace_step = ck["trace_n"], ck["trace_num"], ck["trace_den"], ck["trace_step"]
        norms, vals, k0, el0 = ck["norms"], ck["vals"], ck["k"] + 1, ck["elapsed"]
        print(f"resumed after step {ck['k']}", flush=True)
    t0 = time.time() - el0
    for k in range(k0, n_steps + 1):
        tr = []
        states, it = schwarz.controller_step(models, states, cfg["tol"], cfg["max_iters"], cfg["min_iters"],
                                             trace=tr)
        iters[k - 1] = int(it[0])
        for n, num, den in tr:
            trace_step.append(k)
            trace_n.append(n)
            trace_num.append(float(num[0]))
            trace_den.append(float(den[0]))
        for i, (m, st) in enumerate(zip(models, states)):
            if m.kind == "fom":
                free = m.codes == fem.FREE
                norms[i].append([np.linalg.norm(st["u"][0]), np.linalg.norm(np.where(free, st["v"][0], 0.0)),
                                 np.linalg.norm(np.where(free, st["a"][0], 0.0))])
            else:
                norms[i].append(np.concatenate([st["uh"][0], st["vh"][0]]))
        if k in record:
            for i, nodes in samples.items():
                st = states[i]
                vals[i].append(np.stack([st["u"][0][nodes], st["v"][0][nodes], st["a"][0][nodes]]))
        el = time.time() - t0
        print(f"step {k}/{n_steps} iters {iters[k - 1]} elapsed {el:.0f}s ({el / k:.1f}s/step)", flush=True)
        if k in record or k == n_steps:
            _write(args, cfg, n_steps, k, record, iters, trace_step, trace_n, trace_num, trace_den, norms,
                   samples, vals, el)
        if k % 25 == 0 and k < n_steps:
            os.makedirs(os.path.dirname(ckpt_path), exist_ok=True)
            with open(ckpt_path + ".tmp", "wb") as fh:
                pickle.dump(dict(k=k, states=states, iters=iters[:k].copy(), trace_n=trace_n, trace_num=trace_num,
                                 trace_den=trace_den, trace_step=trace_step, norms=norms, vals=vals, elapsed=el),
                            fh, protocol=5)
            os.replace(ckpt_path + ".tmp", ckpt_path)


def _write(args, cfg, n_steps, k_done, record, iters, trace_step, trace_n, trace_num, trace_den, norms, samples,
           vals, elapsed):
    name = args.out or f"{args.config}_long"
    path = os.path.join(GOLDEN, name + ".npz")
    data = dict(iters=iters[:k_done], record=np.array([r for r in record if r <= k_done], dtype=np.int64),
                trace_step=np.array(trace_step), trace_n=np.array(trace_n), trace_num=np.array(trace_num),
                trace_den=np.array(trace_den), steps_done=np.array(k_done))
    for i, nrm in norms.items():
        data[f"norms_{i}"] = np.array(nrm)
    for i, nodes in samples.items():
        data[f"nodes_{i}"] = nodes
        if vals[i]:
            data[f"values_{i}"] = np.stack(vals[i])     # (n_record, 3 fields u v a, n_sample, 3)
    tmp = path + ".tmp.npz"
    np.savez_compressed(tmp, **data)
    os.replace(tmp, path)
    try:
        rev = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True).stdout.strip()
    except OSError:
        rev = "?"
    prov = dict(script="tools/gen_golden_fullsize.py", config=args.config, steps_requested=n_steps,
                steps_done=int(k_done), record=[int(r) for r in record], git_head=rev, numpy=np.__version__,
                python=platform.python_version(), host=platform.node(), cpu=platform.processor(),
                oracle_seconds=round(elapsed, 1), sample_seed=20251120,
                sha256=hashlib.sha256(open(path, "rb").read()).hexdigest(),
                source="oracle only (oracle.schwarz.controller_step); no value from the CUDA path")
    if getattr(args, "rom_ops_id", None):
        prov["rom_ops_id"] = args.rom_ops_id     # the trained operators this run used (tools/gen_c4_rom.py)
    with open(os.path.join(GOLDEN, name + ".json"), "w") as fh:
        json.dump(prov, fh, indent=1)


if __name__ == "__main__":
    main()
