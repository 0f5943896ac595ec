"""Image-batch partitioning across the GPUs of one box.

The prefix forward is embarrassingly data-parallel over images: eval-mode BN uses
running statistics and no layer mixes images, so each rank runs its own contiguous
shard through ``hapi_prefix_forward`` with no data-path collective.  The paper already
spreads requests "evenly on the existing GPUs" with batch adaptation "separately for each
GPU"; contiguous ranges keep the order, so concatenating the per-rank send
buffers reproduces the single-GPU output (the client's reorder step, becomes
an identity).  The only collective is an all_gather of [count, elapsed_ns, checksum] per
rank for reporting (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank r of R gets images [floor(r*N/R), floor((r+1)*N/R))."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError((n, world, rank))
    return (rank * n) // world, ((rank + 1) * n) // world


def checksum_bits(x: float) -> int:
    """Exact float64 checksum carried as int64 bits through an integer collective."""
    return int(np.float64(x).view(np.int64))


def gather_meta(count: int, elapsed_ns: int, checksum: float, device=None, group=None) -> np.ndarray:
    """all_gather of [count, elapsed_ns, checksum bits] -> int64 array [world, 3]."""
    import torch
    import torch.distributed as dist
    meta = torch.tensor([count, elapsed_ns, checksum_bits(checksum)], dtype=torch.int64, device=device)
    if not (dist.is_available() and dist.is_initialized()):
        return meta.view(1, 3).cpu().numpy()
    world = dist.get_world_size(group)
    out = torch.empty(world * 3, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, meta, group=group)
    return out.view(world, 3).cpu().numpy()


def summarize(meta: np.ndarray):
    """-> (total images, max elapsed seconds over ranks, aggregate img/s, per-rank checksums)."""
    total = int(meta[:, 0].sum())
    tmax = float(meta[:, 1].max()) / 1e9
    checks = [float(np.int64(v).view(np.float64)) for v in meta[:, 2]]
    return total, tmax, (total / tmax if tmax > 0 else 0.0), checks


def run_shard(n_total: int, world: int, rank: int, chunk: int, forward: Callable[[int, int], float]):
    """Process this rank's shard in chunks of `chunk` images; `forward(start, count)` runs one
    chunk and returns its checksum contribution.  Returns (count, checksum)."""
    a, b = shard_range(n_total, world, rank)
    s = 0.0
    for c0 in range(a, b, chunk):
        s += forward(c0, min(chunk, b - c0))
    return b - a, s
