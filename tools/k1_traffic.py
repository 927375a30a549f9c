"""profiles/k1_ncu_summary.json from an `ncu --set full` capture of the 6 K1 launches of one c3 controller step
(host-driven sweeps: Omega_1, Omega_2 of sweeps 1, 2, 3; tools/gpu_round.sh).  bench.py reports the mean DRAM
bytes per launch as roofline.traffic next to the algorithmic bytes of the same launches (DESIGN.md section 6:
96 B per node, plus 24 B per node of the Schwarz band from sweep 2 on, R38)."""
import csv
import json
import subprocess
import sys


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, u = r[0], r[1]
    rows = [x for x in r[2:] if "fom_tiled" in x[h.index("Kernel Name")]]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ns": 1e-3, "ms": 1e3}

    def val(row, name):
        i = h.index(name)
        return float(row[i].replace(",", "")) * scale.get(u[i], 1.0)
    dram = [val(x, "dram__bytes_read.sum") + val(x, "dram__bytes_write.sum") for x in rows]
    us = [val(x, "gpu__time_duration.sum") for x in rows]
    # c3: Omega_1 141x256x256 elements (Schwarz face x+, band = 2 node layers), Omega_2 110x200x200 (x-)
    nodes = [142 * 257 * 257, 111 * 201 * 201]
    band = [2 * 257 * 257, 2 * 201 * 201]
    alg = [96.0 * nodes[i % 2] + (24.0 * band[i % 2] if i >= 2 else 0.0) for i in range(len(rows))]
    d = dict(source=f"ncu --set full of the {len(rows)} K1 launches of one c3 controller step ({rep}, host-driven "
                    "sweeps; Omega_1, Omega_2 of sweeps 1-3)", workload="c3",
             dram_bytes_per_k1_launch=sum(dram) / len(dram), algorithmic_bytes_per_k1_launch=sum(alg) / len(alg),
             per_launch_dram_bytes=dram, per_launch_algorithmic_bytes=alg, per_launch_us=us)
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in d.items() if not k.startswith("per_")}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/k1_ncu_summary.json")
