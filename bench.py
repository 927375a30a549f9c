#!/usr/bin/env python
"""Benchmark of the O-SAM FOM/OpInf coupled time loop on B200 (one JSON line on rank 0).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload c3]

A "step" is one controller step of Algorithm 1 (all Schwarz sweeps until convergence,
every row of SURVEY 8(a)) over the workload.  Default workload: BASELINE config c3
(large FOM-FOM, 41,590,407 DOFs; the largest single-GPU pure-FOM config, on which the
north_star's HBM-roofline target is stated).  `value` = FOM DOF-updates/s summed over all
ranks (every FOM DOF counts once per Schwarz sweep).  N > 1 runs independent
replicas (weak scaling, no data-path collective).
--impl reference times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import osam_inputs as I  # noqa: E402

METRIC = "FOM DOF-updates/s"
UNIT = "DOF-updates/s"
SAMPLE_LATERAL = 32
FALLBACK_HBM = 6650.0
# FP64 CUDA-core peak derived from unit counts and clock: 148 SMs x 64 FP64 FMA/clk
# x 2 flop x 1.965 GHz (clocks.max.sm, B200_PROFILING.md)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# algorithmic FP64 flops of NL1 per element and FOM advance (FMA = 2): 36 edge
# differences + 8 Gauss points x (gradient 72 + stress (SVK 94 / Neohookean 169) + force accumulation 72)
# + 72 nodal assembly
NL1_FLOPS_PER_ELEMENT = {"svk": 36 + 8 * (72 + 94 + 72) + 72, "neohookean": 36 + 8 * (72 + 169 + 72) + 72}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="c3")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-largest", action="store_true", help="skip the c4 (largest config) K1 roofline entry")
    p.add_argument("--material", default="linear", choices=["linear", "svk", "neohookean"],
                   help="FOM material (NEXT-3): nonlinear materials run kernel NL1 (FP64-ALU roofline)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_desc(cfg):
    parts = []
    dofs = 0
    for s in cfg["subdomains"]:
        n = (s["nel"][0] + 1) * (s["nel"][1] + 1) * (s["nel"][2] + 1)
        if s["kind"] == "fom":
            dofs += 3 * n
        extra = f" r={cfg['rom']['r']}" if s["kind"] == "rom" else ""
        parts.append(f"{s['kind'].upper()} {s['nel'][0]}x{s['nel'][1]}x{s['nel'][2]}{extra}")
    return " | ".join(parts), dofs


def sample_cfg(cfg, lateral=SAMPLE_LATERAL):
    """Bounded CPU sample of a FOM workload: same x-structure (meshes, overlap, Schwarz faces,
    BCs, IC, dt), lateral extent cut to `lateral` elements of the first subdomain."""
    out = dict(cfg)
    subs = []
    ref = cfg["subdomains"][0]
    lateral = min(lateral, ref["nel"][1], ref["nel"][2])  # a sample never grows the workload
    for s in cfg["subdomains"]:
        ny = max(1, round(lateral * s["nel"][1] / ref["nel"][1]))
        nz = max(1, round(lateral * s["nel"][2] / ref["nel"][2]))
        hy = s["hi"][1] * lateral / ref["nel"][1]
        hz = s["hi"][2] * lateral / ref["nel"][2]
        subs.append(dict(s, hi=(s["hi"][0], hy, hz), nel=(s["nel"][0], ny, nz)))
    out["subdomains"] = subs
    return out


def workload_ops(cfg):
    """Reduced operators of the ROM subdomains: seeded stand-ins of the trained sizes (the offline
    training runs of c2/c4/c5 are minutes to an hour of CPU work; throughput does not depend on the
    operator values; parity with trained operators is covered by tests/).  None for FOM-only workloads."""
    if not any(s["kind"] == "rom" for s in cfg["subdomains"]):
        return None
    from paper_2511_20687_b200 import problem
    return problem.synthetic_rom_ops(cfg)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_rate(cfg, warmup, steps=None, seconds=None, threads=None):
    """Oracle DOF-updates/s on cfg: `warmup` untimed controller steps then `steps` timed (or
    as many as fit in `seconds`), with `threads` threads in the C element loop and the BLAS pool (None:
    all host cores).  Returns (rate, steps_timed, wall, threads used)."""
    from threadpoolctl import threadpool_limits
    from oracle import cfem
    n_thr = cfem.set_threads(threads or 0)
    with threadpool_limits(limits=n_thr):
        return _oracle_rate(cfg, warmup, steps, seconds) + (n_thr,)


def _oracle_rate(cfg, warmup, steps=None, seconds=None):
    from oracle import schwarz
    ops = workload_ops(cfg)
    from paper_2511_20687_b200 import problem
    models = schwarz.build_models(cfg, rom_ops=ops, e_scale=problem.e_scale(cfg))
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    st = [m.init_state(u) for m, u in zip(models, u0s)]
    dofs = sum(3 * m.box.n_nodes for m in models if m.kind == "fom")
    if dofs == 0:  # ROM-only (c5): reduced updates, r x batch per ROM and sweep
        dofs = sum(m.Kbar.shape[0] * m.batch for m in models if m.kind == "rom")
    for _ in range(warmup):
        st, _ = schwarz.controller_step(models, st, cfg["tol"], cfg["max_iters"], cfg["min_iters"])
    t0 = time.perf_counter()
    n = 0
    sweeps = 0
    while True:
        st, it = schwarz.controller_step(models, st, cfg["tol"], cfg["max_iters"], cfg["min_iters"])
        n += 1
        sweeps += int(it.max())
        el = time.perf_counter() - t0
        if (steps is not None and n >= steps) or (seconds is not None and el >= seconds and n >= 3):
            break
    return sweeps * dofs / el, n, el


def max_over_ranks(x, dist, dev=None):
    """Max of a per-rank float over all ranks (the timing rule: max over ranks); identity at N=1."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, dist, dev=None):
    """Sum of a per-rank float over all ranks (whole-job work); identity at N=1."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


def ncu_traffic():
    """dram bytes per K1 launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "k1_ncu_summary.json")
    try:
        return float(json.load(open(path))["dram_bytes_per_k1_launch"])
    except Exception:
        return None


class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.06)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = I.config(args.workload)
    sample = sample_cfg(cfg)
    desc, _ = workload_desc(cfg)
    sdesc, _ = workload_desc(sample)
    rate, n, el, threads = oracle_rate(sample, args.warmup, steps=args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / n, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {desc}", "sample": sdesc, "parallelism": "rank 0 only"},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"{args.workload} with lateral extent cut to {SAMPLE_LATERAL} elements: {sdesc}; "
                                       f"{n} controller steps after {args.warmup} warm-up"},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def k1_profile(cfg, subs, stream, dev, steps):
    """K1 launch timing: `steps` controller steps in profiling mode (host-driven sweeps, a CUDA event
    pair around every K1 launch on the subdomains' stream).  Returns (profile dict, elapsed ms)."""
    import torch
    from paper_2511_20687_b200 import osam, problem
    osam.set_profiling(True)
    osam.reset_profile()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    problem.run(cfg, subs, n_steps=steps)
    p1.record(stream)
    torch.cuda.synchronize(dev)
    osam.set_profiling(False)
    return osam.get_profile(), p0.elapsed_time(p1)


def roofline_of(prof, prof_ms, peak):
    k1_ms = prof["k1_ms"] / max(1, prof["k1_launches"])
    achieved = prof["k1_bytes"] / max(1, prof["k1_launches"]) / (k1_ms / 1e3) / 1e9
    return {"achieved": achieved, "frac": achieved / peak, "k1_ms_per_launch": k1_ms,
            "k1_share_of_step": prof["k1_ms"] / prof_ms}


def c4_trained_ops():
    """c4's oracle-trained ROMs (tools/gen_c4_rom.py: Phi on the rows the transfer reads, reduced IC), or None."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    try:
        import gen_c4_rom
        return gen_c4_rom.load_online_ops()
    except Exception:
        return None


def largest_config(dev, stream, steps=60, warmup=5):
    """North_star's HBM target is stated on the largest config (c4: 256^3 FOM between two r = 200 ROMs):
    steps/s and the K1 roofline there, measured the same way as the headline (in-schedule K1 timeline).  The
    ROMs are the oracle-trained ones when cache/c4_rom_ops.npz exists, else seeded stand-ins of their sizes."""
    import torch
    from paper_2511_20687_b200 import osam, problem
    cfg = I.config("c4")
    desc, fom_dofs = workload_desc(cfg)
    trained = c4_trained_ops()
    ops = trained if trained is not None else workload_ops(cfg)
    subs = problem.build(cfg, {i: dict(o) for i, o in ops.items()}, stream=stream.cuda_stream)
    fields = problem.initial_fields(cfg)
    for i, (sub, f) in enumerate(zip(subs, fields)):
        if trained is not None and cfg["subdomains"][i]["kind"] == "rom":
            sub.set_ic_reduced(np.ascontiguousarray(ops[i]["uh0"]), None, np.ascontiguousarray(ops[i]["s0"]))
        else:
            sub.set_ic(torch.from_numpy(f).to(dev))
    problem.run(cfg, subs, n_steps=warmup)
    torch.cuda.synchronize(dev)
    osam.k1_timeline(subs, reset=True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, iters = problem.run(cfg, subs, n_steps=steps)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    tl = osam.k1_timeline(subs, reset=True)
    prof, prof_ms = k1_profile(cfg, subs, stream, dev, 10)
    peak, _ = measured_peak()
    achieved = tl["bytes"] / (tl["union_ms"] / 1e3) / 1e9 if tl["union_ms"] > 0 else 0.0
    rs = roofline_of(prof, prof_ms, peak)
    out = {"workload": f"c4: {desc} ({fom_dofs} FOM DOFs; ROM operators: "
                       + ("oracle-trained (tools/gen_c4_rom.py)" if trained is not None else
                          "seeded stand-ins of the trained sizes (cache/c4_rom_ops.npz absent)") + ")",
           "steps": steps, "ms_per_step": ms / steps, "schwarz_steps_per_s": 1e3 * steps / ms,
           "fom_dof_updates_per_s": int(iters.max(axis=1).sum()) * fom_dofs / (ms / 1e3),
           "schwarz_iters_per_step": float(iters.max(axis=1).mean()),
           "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s", "achieved": achieved, "frac": achieved / peak,
                        "k1_busy_ms_per_step": tl["union_ms"] / steps, "k1_share_of_step": tl["union_ms"] / ms,
                        "k1_ms_per_launch": tl["sum_ms"] / max(1, tl["launches"]),
                        "serial_profile": {"achieved": rs["achieved"], "frac": rs["frac"],
                                           "k1_ms_per_launch": rs["k1_ms_per_launch"],
                                           "k1_share_of_step": rs["k1_share_of_step"]}}}
    for sub in subs:
        sub.close()
    return out


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl ours needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2511_20687_b200 import osam, problem

    cfg = I.config(args.workload)
    sharded = world > 1 and cfg.get("batch", 1) > 1
    if sharded:  # c5: the samples are independent problems -> B/N samples per rank (shard.py)
        from paper_2511_20687_b200 import shard
        cfg = shard.shard_cfg(cfg, world, rank)
    if args.material != "linear":
        cfg["material"] = args.material
    desc, fom_dofs = workload_desc(cfg)
    stream = torch.cuda.current_stream(dev)
    trained = c4_trained_ops() if args.workload == "c4" else None
    ops = trained if trained is not None else workload_ops(cfg)
    subs = problem.build(cfg, ops, stream=stream.cuda_stream)
    fields = problem.initial_fields(cfg)
    if trained is not None:  # c4's trained ROMs take the oracle's reduced IC (Phi given on the lift rows only)
        for i, s_ in enumerate(cfg["subdomains"]):
            if s_["kind"] == "rom":
                fields[i] = None
    gpu_fields = [None if f is None else torch.from_numpy(f).to(dev) for f in fields]

    def upload_ic(src):
        for i, (sub, f) in enumerate(zip(subs, src)):
            if f is None:
                sub.set_ic_reduced(np.ascontiguousarray(ops[i]["uh0"]), None, np.ascontiguousarray(ops[i]["s0"]))
            else:
                sub.set_ic(f)

    upload_ic(gpu_fields)
    # warm-up (first call binds the Schwarz maps)
    problem.run(cfg, subs, n_steps=args.warmup)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    clocks = Clocks(local)
    osam.reset_profile()
    osam.k1_timeline(subs, reset=True)
    barrier()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, iters = problem.run(cfg, subs, n_steps=args.steps)  # one CUDA graph per controller step
    e1.record(stream)
    barrier()
    ck = clocks.stop()
    launches = osam.get_profile()["kernel_launches"]
    ms = e0.elapsed_time(e1)
    # K1 roofline in the timed schedule itself: first-CTA-start / last-CTA-end stamps of every K1 launch,
    # folded per sweep on the device (osam_get_k1_timeline)
    tl = osam.k1_timeline(subs, reset=True)
    # serialised per-launch K1 times (comparable with the ncu launch list): the same steps in profiling mode
    prof_steps = max(3, min(args.steps, 30))
    prof, prof_ms = k1_profile(cfg, subs, stream, dev, prof_steps)
    ms = max_over_ranks(ms, dist, dev)
    sweeps = int(iters.max(axis=1).sum())
    value = sum_over_ranks(sweeps * fom_dofs, dist, dev) / (ms / 1e3)
    steps_per_s = args.steps / (ms / 1e3)
    # ROM-only workloads (c5): reduced updates/s = sum over sweeps and ROMs of r * batch
    rom_units = sum(cfg["rom"]["r"] * cfg.get("batch", 1) for s_ in cfg["subdomains"] if s_["kind"] == "rom")
    rom_only = fom_dofs == 0
    if rom_only:
        value = sum_over_ranks(sweeps * rom_units, dist, dev) / (ms / 1e3)

    # end to end through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        host_in = [None if f is None else torch.from_numpy(f).pin_memory() for f in fields]
        # state read-back: FOM u, v (3n each); ROM u^, v^ (r x batch each)
        host_out = [torch.empty(2 * (3 * sub.n_nodes if sub.kind == osam.OSAM_FOM else sub.r * sub.batch),
                                dtype=torch.float64).pin_memory() for sub in subs]
        barrier()
        t0 = time.perf_counter()
        upload_ic(host_in)
        _, it2 = problem.run(cfg, subs, n_steps=args.steps)
        for sub, h in zip(subs, host_out):
            n = h.numel() // 2
            sub.get_state(h[:n], h[n:])
        barrier()
        el = max_over_ranks(time.perf_counter() - t0, dist, dev)
        h2d = sum(f.nbytes for f in fields if f is not None) + sum(
            8 * (ops[i]["uh0"].size + ops[i]["s0"].size) for i, f in enumerate(fields) if f is None)
        d2h = sum(8 * h.numel() for h in host_out) + 4 * int(it2.size)
        e2e = {"value": sum_over_ranks(int(it2.max(axis=1).sum()) * (rom_units if rom_only else fom_dofs), dist,
                                       dev) / el,
               "unit": "reduced updates/s" if rom_only else UNIT,
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "note": "set_ic(pinned host IC) + osam_step(K) + get_state(pinned host u,v) per run; bytes / K"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peak()
    k1_ms_per_launch = prof["k1_ms"] / max(1, prof["k1_launches"])
    bytes_per_launch = prof["k1_bytes"] / max(1, prof["k1_launches"])
    achieved_serial = bytes_per_launch / (k1_ms_per_launch / 1e3) / 1e9 if k1_ms_per_launch > 0 else 0.0
    achieved = tl["bytes"] / (tl["union_ms"] / 1e3) / 1e9 if tl["union_ms"] > 0 else 0.0
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {desc} ({fom_dofs} FOM DOFs)",
                       "l2": ("inputs larger than L2 (two state buffers x (q, w) x 8 B x FOM DOFs, > 126 MB)"
                              if 32 * fom_dofs > 126e6 else
                              "state and operators fit the 126 MB L2 and are not flushed: a latency-bound config, "
                              "L2-resident by design (no HBM roofline claim)"),
                       **({"rom_operators": "oracle-trained (tools/gen_c4_rom.py, cache/c4_rom_ops.npz)" if trained
                           is not None else "seeded stand-ins of the trained sizes (osam_inputs.synthetic_rom_operators)"}
                          if any(s_["kind"] == "rom" for s_ in cfg["subdomains"]) else {}),
                       "parallelism": (f"samples sharded {I.config(args.workload)['batch']}/{world} per rank, no "
                                       "data-path collective" if sharded else "replicas") if world > 1 else "1 GPU"},
            "schwarz_steps_per_s": world * steps_per_s,
            "schwarz_iters_per_step": float(iters.max(axis=1).mean()),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(), "kernel": "K1 fom_advance",
                         "bytes_model": "32 B/DOF/sweep (read q, w; write q, w) + from sweep 2 8 B per DOF within one node layer of a Schwarz face (read previous w'; elsewhere the norm term is exactly 0, DESIGN.md R38), two-vector form (SURVEY 8(d), DESIGN.md R30)",
                         "k1_bytes_per_step": tl["bytes"] / args.steps,
                         "k1_busy_ms_per_step": tl["union_ms"] / args.steps,
                         "k1_ms_per_launch": tl["sum_ms"] / max(1, tl["launches"]),
                         "k1_launches_per_step": tl["launches"] / args.steps,
                         "k1_share_of_step": tl["union_ms"] / ms,
                         # algorithmic bytes per controller step x steps/s / peak
                         "step_frac": tl["bytes"] / args.steps * steps_per_s / 1e9 / peak,
                         "timing": "in the timed region itself: every K1 launch stamps its first CTA start and last "
                                   "CTA end (%globaltimer); K3 folds them per sweep into the time some K1 runs (the "
                                   "union of the concurrent subdomains' launches); achieved = K1 algorithmic bytes / "
                                   "that time, so k1_share_of_step <= 1",
                         "serial_profile": {"k1_ms_per_launch": k1_ms_per_launch, "achieved": achieved_serial,
                                            "frac": achieved_serial / peak, "k1_share_of_step": prof["k1_ms"] / prof_ms,
                                            "timing": f"CUDA events around each K1 over {prof_steps} steps in "
                                                      "profiling mode (host-driven sweeps, K1s serialised on one "
                                                      "stream), as the ncu launch list sees them"},
                         "peak_source": peak_src},
            "gpu_launches": int(launches),
            "clocks": ck, "e2e": e2e}
    if rom_only:  # no FOM: the reduced updates are GEMM-shaped (DMMA when batched) but latency-bound
        line["metric"], line["unit"] = "reduced updates/s", "reduced updates/s"
        ops = workload_ops(cfg)
        flops = 0.0  # per controller step: 2 r (r + r_b) + 2 n_s r_b per sample, ROM and sweep (8(d))
        for i, s_ in enumerate(cfg["subdomains"]):
            if s_["kind"] == "rom":
                r_, rb_ = ops[i]["Kbar"].shape[0], ops[i]["Bbar"].shape[1]
                flops += (2 * r_ * (r_ + rb_) + 2 * ops[i]["Phi_s"].shape[0] * rb_) * cfg.get("batch", 1)
        tf = flops * sweeps / args.steps * steps_per_s / 1e12
        line["roofline"] = {"bound": "tensor", "achieved": tf, "peak": 45.0, "unit": "TFLOP/s", "frac": tf / 45.0,
                            "traffic": None, "kernel": "ROM update + boundary projection (DMMA GEMMs), step level",
                            "note": "latency-bound (GEMMs of r = 400 x 64 samples); peak = B200 FP64 tensor "
                                    "(blackwell_cuda_programming.md); the lift GEMM is not counted",
                            "peak_source": "guide"}
    if args.material != "linear":   # NL1 is FP64-ALU bound: roofline in TFLOP/s
        n_fom = sum(1 for s in cfg["subdomains"] if s["kind"] == "fom")
        elems = sum(int(np.prod(s["nel"])) for s in cfg["subdomains"] if s["kind"] == "fom")
        flops = NL1_FLOPS_PER_ELEMENT[args.material] * elems / max(1, n_fom)   # per launch (mean)
        tf = flops / (k1_ms_per_launch / 1e3) / 1e12
        line["metric"] = METRIC
        line["config"]["workload"] += f", material {args.material}"
        line["roofline"] = {"bound": "alu", "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                            "frac": tf / FP64_PEAK_TFLOPS, "traffic": None, "kernel": "NL1 fom_nl_kernel",
                            "flops_model": f"{NL1_FLOPS_PER_ELEMENT[args.material]} FP64 flop per element per "
                                           "FOM advance (DESIGN.md section 11)",
                            "hbm_achieved_gbs": achieved_serial, "k1_ms_per_launch": k1_ms_per_launch,
                            "k1_share_of_step": prof["k1_ms"] / prof_ms,
                            "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"}
    if world == 1 and not args.no_largest and args.workload != "c4" and args.material == "linear":
        line["largest_config"] = largest_config(dev, stream)
    if world == 1 and not args.no_cpu_baseline:
        sample = sample_cfg(cfg)
        sdesc, _ = workload_desc(sample)
        rate, n, el, threads = oracle_rate(sample, 1, seconds=10.0)
        rate1, n1, el1, _ = oracle_rate(sample, 1, seconds=8.0, threads=1)
        line["cpu_baseline"] = {"value": rate, "unit": line["unit"], "cores": threads, "kind": "oracle",
                                "cpu": cpu_model(), "host_cores": os.cpu_count(),
                                "one_thread": {"value": rate1, "steps": n1, "seconds": round(el1, 1)},
                                "sample": f"{args.workload} with lateral extent cut to {SAMPLE_LATERAL} elements "
                                          f"({sdesc}); {n} controller steps, {el:.1f} s; threads = the C element "
                                          "loop's OpenMP threads and the BLAS pool (the rest of the NumPy loop is "
                                          "single-threaded)"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
