"""GPU long-horizon parity at BASELINE's full sizes (c3 over its 500-step horizon; c4 with trained ROMs),
in the launch configuration bench.py times (CUDA graphs, parallel FOM branches, the tiled K1).

Expected values come from tests/golden/<cfg>_long.npz, written by tools/gen_golden_fullsize.py, which calls
only oracle/ (Algorithm 1 P:L370-404 on the full meshes; the force by the C element loop oracle/cfem.c) and
records: the Schwarz iteration count of every step; the (num, den) pair of every tested iteration
(eq:conv_criterion P:L443-467); per subdomain ||u||, ||v||, ||a|| (FOM) or u^, v^ (ROM) after every step;
a seeded sample of 6000 FOM nodes per subdomain (uniform, within two layers of a Schwarz face, on the
exterior faces, near the pulse, the corners) with u, v, a at the recorded steps.

Bar: identical iteration counts at every step; relative L2 <= 1e-10 of the sampled (u, v, a) per
subdomain and field and of the reduced states; norms to 1e-10; den of the trace to 1e-12, num to 1e-11
(tests/test_gpu_convergence.py explains the cancellation in num), num == 0.0 where the oracle's is.
"""
import json
import os
import sys

import numpy as np
import pytest

import osam_inputs as I

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam, problem
    osam.lib()
    return osam, problem


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def golden(name):
    path = os.path.join(GOLD, f"{name}_long.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/gen_golden_fullsize.py {name})")
    return np.load(path)


def trace_ref(z, n_steps, T):
    out = np.full((n_steps, T, 1, 2), np.nan)
    for k, n, num, den in zip(z["trace_step"], z["trace_n"], z["trace_num"], z["trace_den"]):
        if k <= n_steps:
            out[k - 1, n - 1, 0] = (num, den)
    return out


def run_and_compare(osam, problem, cfg, subs, z):
    n_steps = int(z["steps_done"])
    record = [int(r) for r in z["record"]]
    osam.set_conv_trace(cfg["max_iters"])
    iters, traces = [], []
    done = 0
    worst = {}
    try:
        for cp in sorted(set(record) | {n_steps}):
            _, it = problem.run(cfg, subs, n_steps=cp - done)
            iters.append(it.copy())
            traces.append(osam.get_conv_trace(subs))
            done = cp
            if cp not in record:
                continue
            ri = record.index(cp)
            for i, sub in enumerate(subs):
                if cfg["subdomains"][i]["kind"] == "fom":
                    u, v, a = problem.fom_state(sub, accel=True)
                    nodes = z[f"nodes_{i}"]
                    ref = z[f"values_{i}"][ri]                       # (3 fields, n_sample, 3)
                    for f, got in enumerate((u, v, a)):
                        e = rel(got[nodes], ref[f])
                        worst[(i, f)] = max(worst.get((i, f), 0.0), e)
                        assert e <= 1e-10, (cp, i, "uva"[f], e)
                    nrm = z[f"norms_{i}"][cp - 1]
                    mine = [np.linalg.norm(u), np.linalg.norm(v), np.linalg.norm(a)]
                    for f in range(3):
                        assert abs(mine[f] - nrm[f]) <= 1e-10 * nrm[f], (cp, i, f, mine[f], nrm[f])
                else:
                    uh, vh = problem.rom_state(sub)
                    r = uh.shape[1]
                    ref = z[f"norms_{i}"][cp - 1]
                    for f, got in enumerate((uh[0], vh[0])):
                        e = rel(got, ref[f * r:(f + 1) * r])
                        worst[(i, f)] = max(worst.get((i, f), 0.0), e)
                        assert e <= 1e-10, (cp, i, f, e)
    finally:
        osam.set_conv_trace(0)
    iters = np.concatenate(iters)[:, 0]
    assert np.array_equal(iters, z["iters"][:n_steps]), "Schwarz iteration counts differ from the oracle's"
    tr = np.concatenate(traces)
    ref = trace_ref(z, n_steps, cfg["max_iters"])
    tested = ~np.isnan(ref[..., 1])
    assert np.array_equal(tested, ~np.isnan(tr[..., 1]))
    num, den, num_r, den_r = tr[..., 0][tested], tr[..., 1][tested], ref[..., 0][tested], ref[..., 1][tested]
    assert np.all(np.abs(den - den_r) <= 1e-12 * den_r)
    zero = num_r == 0.0
    assert np.array_equal(num[zero], num_r[zero])
    assert np.all(np.abs(num[~zero] - num_r[~zero]) <= 1e-11 * num_r[~zero])
    print(f"{cfg['name']}: {n_steps} steps, iterations {np.unique(iters).tolist()}, worst rel L2 per (subdomain, "
          f"field) {({k: float(f'{v:.2e}') for k, v in worst.items()})}")


def test_c3_full_size_long_horizon(gpu):
    osam, problem = gpu
    z = golden("c3")
    cfg = I.config("c3")
    subs = problem.build(cfg)
    problem.set_ics(cfg, subs, device="cuda:0")
    run_and_compare(osam, problem, cfg, subs, z)


def c4_online_ops():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_c4_rom
    ops = gen_c4_rom.load_online_ops()
    if ops is None:
        pytest.skip("cache/c4_rom_ops.npz not generated (tools/gen_c4_rom.py)")
    return ops


def test_c4_full_size_trained_roms(gpu):
    """c4 with the oracle-trained r = 200 ROMs (Phi given on the rows the transfer reads, reduced IC)."""
    osam, problem = gpu
    z = golden("c4")
    ops = c4_online_ops()
    import gen_c4_rom
    with open(os.path.join(GOLD, "c4_long.json")) as fh:
        want = json.load(fh).get("rom_ops_id")
    if want is not None and gen_c4_rom.rom_ops_id(ops) != want:
        pytest.skip("cache/c4_rom_ops.npz comes from another training run than tests/golden/c4_long.npz "
                    "(rerun tools/gen_golden_fullsize.py c4)")
    cfg = I.config("c4")
    subs = problem.build(cfg, {i: dict(o) for i, o in ops.items()})
    for i, sub in enumerate(subs):
        if cfg["subdomains"][i]["kind"] == "rom":
            sub.set_ic_reduced(np.ascontiguousarray(ops[i]["uh0"]), None, np.ascontiguousarray(ops[i]["s0"]))
        else:
            sub.set_ic(problem.initial_fields(cfg)[i])
    run_and_compare(osam, problem, cfg, subs, z)
