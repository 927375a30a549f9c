"""GPU: the runtime switches that are read once per process (OSAM_SERIAL_K1: FOM advances on the main stream;
OSAM_PDL=0: no programmatic dependent launch; OSAM_NOGRAPH=1: host-driven sweeps) keep the results.  Each runs in
a subprocess on two cases -- scaled c3 (the tiled K1 of two subdomains, several tiles and z-chunks) and the scaled
c4 topology with trained ROMs (the ROM chain between FOM advances) -- compared with the oracle at the parity bar
(1e-10, identical iteration counts; tests/test_gpu_parity.py run_both).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch
assert torch.cuda.is_available()
import osam_inputs as I
from oracle import opinf
from test_gpu_parity import run_both
from paper_2511_20687_b200 import problem
cfg = I.scaled(I.config("c3"), 8.0)
_, it, worst = run_both(problem, cfg, 12, checkpoints=(1,))
assert (it == 3).all()
cfg = I.scaled(I.config("c4"), 10.0)
cfg["rom"] = dict(cfg["rom"], r=40)
cfg["rom"]["training"] = dict(cfg["rom"]["training"], n_steps=120,
                              subdomains=[dict(s, kind="fom", nel=(8, 8, 8)) for s in cfg["subdomains"]])
for s in cfg["subdomains"]:
    if s["kind"] == "rom":
        s["nel"] = (8, 8, 8)
_, it2, worst2 = run_both(problem, cfg, 15, rom_ops=opinf.train(cfg, I), checkpoints=(1,))
print("ok", worst, worst2)
'''


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("env", [{"OSAM_SERIAL_K1": "1"}, {"OSAM_PDL": "0"}, {"OSAM_NOGRAPH": "1"},
                                 {"OSAM_XFER_INGRID": "1"}, {"OSAM_XFER_PIPE": "0"}, {"OSAM_UNROLL_MIN": "0"}])
def test_process_wide_switches_keep_parity(gpu, env):
    e = dict(os.environ, OSAM_GATHER_MAX="0", **env)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert out.stdout.strip().splitlines()[-1].startswith("ok")


ROM_SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch
assert torch.cuda.is_available()
import osam_inputs as I
from oracle import opinf
from test_gpu_parity import run_both
from paper_2511_20687_b200 import problem
cfg = I.config("c2")
_, it, worst = run_both(problem, cfg, 120, rom_ops=opinf.train(cfg, I), checkpoints=(1,))
assert (it == 3).all()
cfg = I.config("c5")
_, it2, worst2 = run_both(problem, cfg, 150, rom_ops=opinf.train(cfg, I), checkpoints=(1,))
assert (it2 == 3).all()
print("ok", worst, worst2)
'''


@pytest.mark.parametrize("env", [{}, {"OSAM_NO_FOLD": "1"}, {"OSAM_ROM_PAR": "0"}, {"OSAM_ROM_KBG": "0"},
                                 {"OSAM_EPI_FUSED": "0"}, {"OSAM_UNROLL_MIN": "0"}])
def test_rom_exchange_switches_keep_parity(gpu, env):
    """c2 (FOM-ROM, B = 1: the FOM exchange folded into the ROM update by default) and c5 (batched ROM-ROM: the
    predictor once per step, parallel ROM branches, [-Kbar | Bbar G] by default) against the oracle, with every
    ROM-exchange switch: OSAM_NO_FOLD=1 (transfer + projection + update), OSAM_ROM_PAR=0 (serial ROM chain, the
    predictor per sweep), OSAM_ROM_KBG=0 (g^ = G u^ before the update GEMM)."""
    e = dict(os.environ, **env)
    code = ROM_SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert out.stdout.strip().splitlines()[-1].startswith("ok")
