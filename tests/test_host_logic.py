"""CPU checks of host-side logic around the CUDA path (no GPU): DOF bookkeeping of the binding,
stand-in operator generation, bench.py helpers, and the N > 1 paths of bench.py on gloo."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, schwarz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _configs():
    out = [I.config(n) for n in ("c1", "c2", "c5")]
    out.append(I.scaled(I.config("c3"), 10.0))
    out.append(I.scaled(I.config("c4"), 16.0))
    return out


@pytest.mark.parametrize("cfg", _configs(), ids=lambda c: c["name"])
def test_dof_split_matches_oracle_codes(cfg):
    """problem.dof_split (product-side sizing of stand-in ROM operators) agrees with the oracle's
    Schwarz-face detection and DOF codes (readings R12, R13)."""
    from paper_2511_20687_b200 import problem
    boxes = [fem.Box(s["lo"], s["hi"], s["nel"]) for s in cfg["subdomains"]]
    faces = schwarz.detect_schwarz_faces(boxes)
    for i, s in enumerate(cfg["subdomains"]):
        codes = fem.dof_codes(boxes[i], s["dirichlet"], faces[i].keys()).reshape(-1)
        assert problem.dof_split(cfg, i) == (int((codes == fem.FREE).sum()), int((codes == fem.SCHWARZ).sum()))


def test_synthetic_rom_operators_shapes_and_seed():
    a = I.synthetic_rom_operators(5000, 300, 20, 7, 1e-6, seed=3)
    b = I.synthetic_rom_operators(5000, 300, 20, 7, 1e-6, seed=3)
    assert a["Phi"].shape == (5000, 20) and a["Phi_s"].shape == (300, 7)
    assert a["Kbar"].shape == (20, 20) and a["Bbar"].shape == (20, 7)
    for k in a:
        assert np.array_equal(a[k], b[k])
    G = a["Phi"].T @ a["Phi"]
    assert np.allclose(np.diag(G), 1.0) and np.abs(G - np.eye(20)).max() < 0.1   # nearly orthonormal
    w = np.sqrt(np.diag(a["Kbar"])) * 1e-6
    assert w.max() < 2.0                                                            # below the explicit limit


def test_bench_workload_sizes_and_sample():
    sys.path.insert(0, ROOT)
    import bench
    desc, dofs = bench.workload_desc(I.config("c3"))
    assert dofs == 41590407                                   # reading R24: the meshes are authoritative
    _, dofs4 = bench.workload_desc(I.config("c4"))
    assert dofs4 == 3 * 257 ** 3
    s = bench.sample_cfg(I.config("c3"))
    assert [x["nel"][0] for x in s["subdomains"]] == [141, 110]
    assert max(x["nel"][1] for x in s["subdomains"]) <= 32
    s1 = bench.sample_cfg(I.config("c1"))                     # never grows a small workload
    assert [x["nel"] for x in s1["subdomains"]] == [x["nel"] for x in I.config("c1")["subdomains"]]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _max_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    q.put((rank, bench.max_over_ranks(1.5 + rank, dist)))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_max_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got == {0: 2.5, 1: 2.5}


def test_reference_arm_under_torchrun_rank0_prints_once():
    """--impl reference under torchrun (N = 2, CPU): rank 0 alone times the oracle and prints one line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--workload", "c1", "--gpus", "2", "--steps", "2", "--warmup", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


# ---- multi-GPU sample sharding of c5 (paper_2511_20687_b200/shard.py) -------------------

def test_sample_slice_partitions_the_batch():
    from paper_2511_20687_b200 import shard
    for B in (1, 5, 63, 64):
        for world in (1, 2, 3, 4, 8):
            if world > B:
                continue
            parts = [shard.sample_slice(B, world, q) for q in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    cfg = I.config("c5")
    s = shard.shard_cfg(cfg, 4, 3)
    assert s["batch"] == 16 and s["samples"]["E"] == cfg["samples"]["E"][48:64]
    with pytest.raises(ValueError):
        shard.shard_cfg(I.config("c3"), 2, 0)


def _c5_small(n_steps=6, r=24):
    """c5 geometry and samples with seeded stand-in operators of rank r (cheap; the sharding is what is tested)."""
    from paper_2511_20687_b200 import problem
    cfg = I.config("c5")
    cfg["rom"] = dict(cfg["rom"], r=r)
    cfg["n_steps"] = n_steps
    ops = {}
    for i in range(2):
        n_free, n_s = problem.dof_split(cfg, i)
        o = I.synthetic_rom_operators(n_free, n_s, r, 6, cfg["dt"], 11 + i)
        ops[i] = o
    return cfg, ops


def _oracle_samples(cfg, ops):
    from oracle import schwarz
    e = np.asarray(cfg["samples"]["E"]) / cfg["E"]
    models = schwarz.build_models(cfg, rom_ops=ops, e_scale=e)
    states, iters = schwarz.run(models, [I.initial_displacements(cfg, s) for s in cfg["subdomains"]], cfg["dt"],
                                cfg["n_steps"], cfg["tol"])
    return np.concatenate([states[0]["uh"], states[0]["vh"], states[1]["uh"], states[1]["vh"]], axis=1), iters.T


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2511_20687_b200 import shard
    cfg, ops = _c5_small()
    mine = shard.shard_cfg(cfg, world, rank)
    st, it = _oracle_samples(mine, ops)
    allst = shard.gather_samples(st, dist, cfg["batch"], world)
    allit = shard.gather_samples(it.astype(np.int64), dist, cfg["batch"], world)
    if rank == 0:
        q.put((allst, allit))
    dist.destroy_process_group()


def test_c5_sample_shards_gloo_world2_equal_the_full_batch():
    """Each rank advances its own slice of the 64 samples (no data-path collective), the per-sample results
    gathered after the run equal the single-process run of the whole batch (oracle on both sides: the library
    needs a GPU; tests/test_gpu_shard.py runs the same split through libosam.so)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allst, allit = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
    cfg, ops = _c5_small()
    st, it = _oracle_samples(cfg, ops)
    assert allst.shape == st.shape == (64, 4 * 24)
    assert np.array_equal(allit, it)
    assert np.abs(allst - st).max() <= 1e-13 * np.abs(st).max()
