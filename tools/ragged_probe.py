"""K1 efficiency vs x-raggedness: c3's subdomains (142 / 111 nodes in x: last 32-wide tile column 14 / 15 wide)
against the same y-z size with x extents that fill every tile column (160 / 128 nodes).  Profiling mode (K1
events), algorithmic bytes / time."""
import copy
import json
import sys

import torch

sys.path.insert(0, ".")
import osam_inputs as I  # noqa: E402
from paper_2511_20687_b200 import osam, problem  # noqa: E402


def k1(cfg, steps=10):
    subs = problem.build(cfg)
    problem.set_ics(cfg, subs, device="cuda:0")
    problem.run(cfg, subs, n_steps=3)
    osam.set_profiling(True)
    osam.reset_profile()
    problem.run(cfg, subs, n_steps=steps)
    torch.cuda.synchronize()
    osam.set_profiling(False)
    p = osam.get_profile()
    for s in subs:
        s.close()
    return p["k1_bytes"] / (p["k1_ms"] / 1e3) / 1e9, p["k1_ms"] / p["k1_launches"]


base = I.config("c3")
full = copy.deepcopy(base)
full["subdomains"][0] = dict(full["subdomains"][0], nel=(159, 256, 256), hi=(159 / 141 * 0.55, 1, 1))
full["subdomains"][1] = dict(full["subdomains"][1], nel=(127, 200, 200), lo=(159 / 141 * 0.55 - 0.1, 0, 0),
                             hi=(159 / 141 * 0.55 - 0.1 + 127 / 110 * 0.55, 1, 1))
for name, cfg in (("c3 (142/111 nodes in x)", base), ("full columns (160/128)", full)):
    gbs, ms = k1(cfg)
    print(json.dumps({"case": name, "k1_gbs": gbs, "frac": gbs / 6552, "k1_ms_per_launch": ms}))
