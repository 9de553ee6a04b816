"""Multi-GPU plumbing: one process per GPU (torchrun), reads sharded across
ranks, every rank holding a full index replica.  The path has no exchange
step, so the only collectives are host-side plumbing outside the data path:
gathering per-read results into input order and max-reducing timings
(the reference's only parallelism is threads over reads,
REF src/driver.cpp:99-142).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [begin, end) of n reads for rank."""
    base, extra = divmod(n, world)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


def align_sharded(align_fn: Callable[[np.ndarray, np.ndarray], np.ndarray], bases: np.ndarray,
                  offsets: np.ndarray, rank: int, world: int, result_dtype: np.dtype,
                  device=None) -> np.ndarray:
    """Align this rank's shard with align_fn(bases, offsets) and all-gather the
    results into input order on every rank."""
    import torch
    import torch.distributed as dist

    n = offsets.size - 1
    b, e = shard_range(n, rank, world)
    ob, oe = int(offsets[b]), int(offsets[e])
    local = align_fn(np.ascontiguousarray(bases[ob:oe]), offsets[b:e + 1] - offsets[b])
    if world == 1:
        return local
    itemsize = np.dtype(result_dtype).itemsize
    mx = max(shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world))
    buf = np.zeros(mx * itemsize, np.uint8)
    buf[:local.nbytes] = local.view(np.uint8)
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    out = np.empty(n, result_dtype)
    for r, p in enumerate(parts):
        rb, re_ = shard_range(n, r, world)
        out[rb:re_] = p.cpu().numpy()[:(re_ - rb) * itemsize].view(result_dtype)
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing over all ranks (timings are reported as the max)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
