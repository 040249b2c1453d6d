"""Multi-process plumbing (one process per GPU, torch.distributed).

The interior blocks of the MSC preconditioner are independent (SURVEY
§8(e)); a sharded apply exchanges one n_g interface vector (all-reduce of the
per-rank F_r z1_r partials), a sharded SpMV of C one more.  `bench.py --gpus
N` shards the blocks with `shard_blocks` (libmscg `mscg_precond_*_shard`);
these helpers are the rank-level pieces the bench uses and the tests exercise
with the gloo backend on CPU.
"""
from __future__ import annotations

import os

import numpy as np


def env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device=None):
    """Initialise the default process group over 127.0.0.1 (container
    hostnames may not resolve)."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    if backend == "nccl" and device is not None:
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group(backend)
    return dist


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Device-timed quantities are reported as the max over ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_blocks(block_rows, world: int) -> list[tuple[int, int]]:
    """Contiguous block ranges per rank, balanced by rows (a proxy for
    factor bytes).  Every rank gets at least one block when possible."""
    rows = np.asarray(block_rows, dtype=np.int64)
    nb = len(rows)
    if world < 1:
        raise ValueError("world must be >= 1")
    if nb == 0:
        return [(0, 0)] * world
    cum = np.concatenate([[0], np.cumsum(rows)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        b = max(bounds[-1] + (1 if bounds[-1] < nb else 0), min(b, nb - (world - r)))
        bounds.append(min(max(b, bounds[-1]), nb))
    bounds.append(nb)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]
