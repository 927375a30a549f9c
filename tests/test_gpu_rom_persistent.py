"""GPU: the persistent controller of batched tensor-core ROM groups (c5; kernels_rom_tc.cu rom_persistent_kernel)
against the per-step CUDA-graph path (OSAM_ROM_PERSIST=0) and the oracle.

The persistent kernel computes the folded boundary input as one dot product per (row, sample) instead of a
split-K GEMM, and forms the norm partials per 32-row tile in the update GEMM's last split: the same arithmetic in
another summation order, so states agree with the graph path to rounding (1e-12 relative per sample and field),
the iteration counts exactly, the trace's den to 1e-12 and num to 1e-10; the oracle comparison of the full c5
horizon on the default (graph) path is tests/test_gpu_parity.py::test_c5_batched_rom_rom; the persistent path is
opt-in (OSAM_ROM_PERSIST=1, measured slower on c5: 6.2k vs 6.8k steps/s, profiles/r3_c5_persistent.log).
"""
import numpy as np
import pytest

import osam_inputs as I
from oracle import opinf, schwarz

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam, problem
    osam.lib()
    return osam, problem


@pytest.fixture(scope="module")
def c5_ops():
    return opinf.train(I.config("c5"), I)


def run(osam, problem, cfg, ops, steps, chunks):
    subs = problem.build(cfg, ops)
    problem.set_ics(cfg, subs, device="cuda:0")
    osam.set_conv_trace(cfg["max_iters"])
    its, trs = [], []
    try:
        for n in chunks:   # several osam_step calls: odd step counts exercise the host-side role flip
            _, it = problem.run(cfg, subs, n_steps=n)
            its.append(it.copy())
            trs.append(osam.get_conv_trace(subs))
    finally:
        osam.set_conv_trace(0)
    st = [problem.rom_state(s, accel=True) for s in subs]
    return np.concatenate(its), np.concatenate(trs), st


def test_c5_persistent_equals_graph(gpu, c5_ops, monkeypatch):
    osam, problem = gpu
    cfg = I.config("c5")
    chunks = (1, 37, 62)
    monkeypatch.setenv("OSAM_ROM_PERSIST", "1")
    it_p, tr_p, st_p = run(osam, problem, cfg, c5_ops, sum(chunks), chunks)
    monkeypatch.setenv("OSAM_ROM_PERSIST", "0")
    it_g, tr_g, st_g = run(osam, problem, cfg, c5_ops, sum(chunks), chunks)
    assert np.array_equal(it_p, it_g) and (it_p == 3).all()
    tested = ~np.isnan(tr_g[..., 1])
    assert np.array_equal(tested, ~np.isnan(tr_p[..., 1]))
    num_p, den_p, num_g, den_g = tr_p[..., 0][tested], tr_p[..., 1][tested], tr_g[..., 0][tested], tr_g[..., 1][tested]
    assert np.all(np.abs(den_p - den_g) <= 1e-12 * den_g)
    zero = num_g == 0.0
    assert np.array_equal(num_p[zero], num_g[zero])
    assert np.all(np.abs(num_p[~zero] - num_g[~zero]) <= 1e-10 * num_g[~zero])
    for a, b in zip(st_p, st_g):
        for x, y in zip(a, b):
            err = np.linalg.norm(x - y, axis=1) / np.linalg.norm(y, axis=1)
            assert err.max() <= 1e-12, err.max()


def test_c5_persistent_against_oracle_with_max_iters_cap(gpu, c5_ops, monkeypatch):
    """max_iters = 2 on the persistent path: every step stops at the cap (OSAM_WNOTCONVERGED), counts and states
    as the oracle's (reading R9: the last iterate is kept)."""
    osam, problem = gpu
    monkeypatch.setenv("OSAM_ROM_PERSIST", "1")
    cfg = I.config("c5")
    n = 20
    subs = problem.build(cfg, c5_ops)
    problem.set_ics(cfg, subs, device="cuda:0")
    rc, iters = problem.run(cfg, subs, n_steps=n, max_iters=2)
    assert rc == 1 and (iters == 2).all()
    e = np.asarray(cfg["samples"]["E"]) / cfg["E"]
    models = schwarz.build_models(cfg, rom_ops=c5_ops, e_scale=e)
    states, it_ref = schwarz.run(models, [I.initial_displacements(cfg, s) for s in cfg["subdomains"]], cfg["dt"], n,
                                 cfg["tol"], max_iters=2)
    assert np.array_equal(it_ref.T, iters.T)
    for sub, st in zip(subs, states):
        uh, vh = problem.rom_state(sub)
        for got, ref in ((uh, st["uh"]), (vh, st["vh"])):
            err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
            assert err.max() <= 1e-10, err.max()
