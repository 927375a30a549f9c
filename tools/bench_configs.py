#!/usr/bin/env python
"""Throughput of the latency-bound BASELINE configs (c1, c2, c5) on one GPU, graph mode.

Not the driver's bench line (bench.py times c3); a measurement aid for DESIGN.md / BASELINE.md.
ROM operators are the seeded stand-ins of bench.py (trained operators are used by the parity tests).
Prints one JSON line per config.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import osam_inputs as I  # noqa: E402
from paper_2511_20687_b200 import osam, problem  # noqa: E402


def measure(name, steps, warmup=20):
    cfg = I.config(name)
    t0 = time.time()
    ops = problem.synthetic_rom_ops(cfg) if "rom" in cfg else None
    t_train = time.time() - t0
    stream = torch.cuda.current_stream()
    subs = problem.build(cfg, ops, stream=stream.cuda_stream)
    problem.set_ics(cfg, subs, device="cuda:0")
    problem.run(cfg, subs, n_steps=warmup)
    torch.cuda.synchronize()
    osam.reset_profile()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, iters = problem.run(cfg, subs, n_steps=steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fom = sum(3 * (s["nel"][0] + 1) * (s["nel"][1] + 1) * (s["nel"][2] + 1) for s in cfg["subdomains"]
              if s["kind"] == "fom")
    sweeps = int(iters.max(axis=1).sum())
    out = dict(workload=name, steps=steps, ms_per_step=ms / steps, schwarz_steps_per_s=1e3 * steps / ms,
               fom_dof_updates_per_s=1e3 * sweeps * fom / ms, iters_per_step=float(iters.max(axis=1).mean()),
               batch=cfg.get("batch", 1), kernel_launches=osam.get_profile()["kernel_launches"],
               offline_training_s=round(t_train, 1), rom_tc=os.environ.get("OSAM_ROM_TC", "default"))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["c1", "c2", "c5"]
    for n in names:
        measure(n, steps=int(os.environ.get("STEPS", "400")))
