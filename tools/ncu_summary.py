"""Summarise ncu outputs: launch list CSV -> per-kernel time shares; .ncu-rep -> key raw metrics."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0].split("::")[-1]
            v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else (1.0 if d["Metric Unit"] == "us" else 1e3))
            agg[k][0] += 1
            agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{v[0]:6d} launches {v[1]:12.1f} us total {v[1]/v[0]:10.2f} us/launch {100*v[1]/tot:6.2f}%  {k}")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_branch.sum",
        "smsp__sass_inst_executed_op_local_st.sum", "sm__inst_executed.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, u = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0].split("::")[-1]
        out.append(f"== {name}")
        for w in WANT:
            if w in h:
                out.append(f"   {w} = {row[h.index(w)]} {u[h.index(w)]}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"### {p}")
        print(launches(p) if p.endswith(".csv") else raw(p))
