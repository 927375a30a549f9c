"""GPU: the c5 sample shards (paper_2511_20687_b200/shard.py) through libosam.so.

On the multi-GPU path each rank runs its slice of the 64 samples as its own batched group.  Here the slices
run one after another on the one GPU of this pool (no rank waits on another, so this is the same
computation), and the per-sample states and iteration counts must equal the full 64-sample run (relative
L2 <= 1e-12 per sample: the batched DMMA GEMMs tile over the sample columns, the split-K order does not
depend on the batch width, so the results agree to rounding), and the oracle on the same inputs.
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
    from paper_2511_20687_b200 import osam, problem, shard
    osam.lib()
    return problem, shard


@pytest.fixture(scope="module")
def c5_ops():
    return opinf.train(I.config("c5"), I)


def run(problem, cfg, ops, n):
    subs = problem.build(cfg, ops)
    problem.set_ics(cfg, subs, device="cuda:0")
    _, iters = problem.run(cfg, subs, n_steps=n)
    states = [problem.rom_state(s) for s in subs]
    return np.concatenate([states[0][0], states[0][1], states[1][0], states[1][1]], axis=1), iters.T.copy()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_c5_shards_equal_full_batch(gpu, c5_ops, world):
    problem, shard = gpu
    cfg = I.config("c5")
    n = 120
    full, it_full = run(problem, cfg, c5_ops, n)
    parts, its = [], []
    for rank in range(world):
        st, it = run(problem, shard.shard_cfg(cfg, world, rank), c5_ops, n)
        parts.append(st)
        its.append(it)
    got = np.concatenate(parts)
    assert np.array_equal(np.concatenate(its), it_full)
    err = np.linalg.norm(got - full, axis=1) / np.linalg.norm(full, axis=1)
    assert err.max() <= 1e-12, err.max()
    if world == 2:   # and the oracle on the same split
        e = np.asarray(cfg["samples"]["E"]) / cfg["E"]
        models = schwarz.build_models(cfg, rom_ops=c5_ops, e_scale=e)
        states, it_ref = schwarz.run(models, [I.initial_displacements(cfg, s) for s in cfg["subdomains"]], cfg["dt"],
                                     n, cfg["tol"])
        ref = np.concatenate([states[0]["uh"], states[0]["vh"], states[1]["uh"], states[1]["vh"]], axis=1)
        assert np.array_equal(it_ref.T, it_full)
        for a, b in ((got, ref),):
            for blk in range(4):
                sl = slice(blk * 400, (blk + 1) * 400)
                e_ = np.linalg.norm(a[:, sl] - b[:, sl], axis=1) / np.linalg.norm(b[:, sl], axis=1)
                assert e_.max() <= 1e-10, (blk, e_.max())
