"""Multi-GPU plumbing: SURVEY 8(e)'s natural split of the batched multi-query workload (config c5).

The 64 samples of c5 (E_b, A_b; BASELINE configs[4]) are independent problems: every controller step, Schwarz
iteration and convergence test is per sample (reading R29), so they shard across ranks with no data-path
collective -- rank q runs the contiguous slice samples[start:stop] as its own batched osam_step group on its
own GPU (one process per GPU, torch.distributed for the plumbing only).  The multiplicative sweep itself is
sequential across subdomains, so a single coupled problem does not shard (c1-c4 run replicas).

Marshalling only: slicing the sample list and gathering per-sample results (outside any timed region).
"""
from __future__ import annotations

import copy

import numpy as np


def sample_slice(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of `batch` samples over `world` ranks: ranks < batch % world take one extra."""
    if not (0 <= rank < world) or world < 1:
        raise ValueError("bad rank / world")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_cfg(cfg: dict, world: int, rank: int) -> dict:
    """The workload restricted to this rank's samples (E_b, A_b sliced; batch = slice length)."""
    out = copy.deepcopy(cfg)
    B = cfg.get("batch", 1)
    if B <= 1 or "samples" not in cfg:
        raise ValueError("only batched multi-sample workloads shard (c5)")
    lo, hi = sample_slice(B, world, rank)
    if hi <= lo:
        raise ValueError(f"rank {rank} of {world} has no sample (batch {B})")
    out["samples"] = {k: tuple(v[lo:hi]) for k, v in cfg["samples"].items()}
    out["batch"] = hi - lo
    out["shard"] = dict(world=world, rank=rank, start=lo, stop=hi, batch=B)
    return out


def gather_samples(local: np.ndarray, dist, batch: int, world: int) -> np.ndarray | None:
    """All per-sample rows (axis 0 = this rank's samples) gathered in sample order on every rank, through
    torch.distributed (gloo or nccl CPU/GPU tensors); `local` may hold 0 rows only if the rank has no sample."""
    import torch
    lo, hi = [], []
    for q in range(world):
        a, b = sample_slice(batch, world, q)
        lo.append(a)
        hi.append(b)
    t = torch.from_numpy(np.ascontiguousarray(local))
    rows = max(b - a for a, b in zip(lo, hi))
    pad = torch.zeros((rows,) + tuple(t.shape[1:]), dtype=t.dtype)
    pad[:t.shape[0]] = t
    if dist.get_backend() == "nccl":
        pad = pad.cuda()
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return np.concatenate([p.cpu().numpy()[:b - a] for p, a, b in zip(parts, lo, hi)], axis=0)
