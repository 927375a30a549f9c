"""GPU: the Schwarz transfer evaluated by the first CTAs of the destination's tiled K1 ("the transfer
in the K1 grid"; opt-in OSAM_XFER_INGRID=1, measured slower) against separate transfer launches (the default).  Same arithmetic in the same
order, so the states must be bitwise equal with identical iteration counts -- on scaled c3 (two tiled FOMs, each
the other's source; Omega1's Schwarz face at x = nx, Omega2's at x = 0) and scaled c4 (the centre FOM fed by two
ROM lifts, the excluded last x column behind the in-grid transfer).  The oracle parity of the default path is in
tests/test_gpu_parity.py and tests/test_gpu_switches.py.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, {root!r})
import torch
assert torch.cuda.is_available()
import osam_inputs as I
from paper_2511_20687_b200 import problem
out = {{}}
for name, scale, n in (("c3", 8.0, 12), ("c4", 4.0, 10)):
    cfg = I.scaled(I.config(name), scale)
    ops = problem.synthetic_rom_ops(cfg) if "rom" in cfg else None
    subs = problem.build(cfg, ops)
    problem.set_ics(cfg, subs, device="cuda:0")
    _, it = problem.run(cfg, subs, n_steps=n)
    out[name + "_iters"] = np.asarray(it)
    for k, (s, sd) in enumerate(zip(subs, cfg["subdomains"])):
        st = problem.fom_state(s) if sd["kind"] == "fom" else problem.rom_state(s)
        for q, a in enumerate(st):
            out[f"{{name}}_{{k}}_{{q}}"] = np.asarray(a)
np.savez({path!r}, **out)
print("ok")
'''


def _run(env, path):
    e = dict(os.environ, OSAM_GATHER_MAX="0", **env)
    code = SCRIPT.format(root=ROOT, path=path)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return dict(np.load(path))


def test_ingrid_transfer_bitwise_equals_separate_launches(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _run({"OSAM_XFER_INGRID": "1"}, str(tmp_path / "ingrid.npz"))
    b = _run({}, str(tmp_path / "separate.npz"))
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert (a["c3_iters"] == 3).all()


def test_pipelined_transfers_bitwise_equal_head_of_sweep_transfers(tmp_path):
    """Default: the transfers into a FOM for sweep n + 1 follow its own advance of sweep n on its branch (DESIGN.md
    §6, "pipelined transfers"); OSAM_XFER_PIPE=0 launches them at the head of their sweep.  Same kernels, same
    values: bitwise equal states and identical counts, in graph mode and with host-driven sweeps."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _run({}, str(tmp_path / "pipe.npz"))
    b = _run({"OSAM_XFER_PIPE": "0"}, str(tmp_path / "head.npz"))
    c = _run({"OSAM_NOGRAPH": "1"}, str(tmp_path / "pipe_host.npz"))
    assert a.keys() == b.keys() == c.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
        assert np.array_equal(a[k], c[k]), k
    assert (a["c3_iters"] == 3).all()
