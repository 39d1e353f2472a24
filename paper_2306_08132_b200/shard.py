"""Multi-GPU partitioning for batched grasp search.

Candidates (and, for multi-object batches, objects) are independent, so the
search shards with NO collective in the optimizer loop: each rank runs the
fused kernel on its own contiguous candidate range; results are gathered once
at the end (fixed-size records: q, losses, status). Per-candidate math does not
depend on the shard, so results are identical for any rank count.
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of `total` items for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def object_major(n_objects: int, per_object: int, world: int, rank: int) -> list[tuple[int, int, int]]:
    """Config 4/5: whole objects per rank so each GPU's SDF grids stay
    L2-resident; returns [(object, cand_lo, cand_hi)] for this rank."""
    olo, ohi = shard_range(n_objects, world, rank)
    return [(o, 0, per_object) for o in range(olo, ohi)]


def gather_rows(local: np.ndarray, total: int, world: int, rank: int, group=None) -> np.ndarray | None:
    """Concatenate every rank's rows in candidate order on rank 0 (torch.distributed,
    any backend: gloo on CPU, nccl on GPU). Returns None on other ranks."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    lo, hi = shard_range(total, world, rank)
    assert local.shape[0] == hi - lo
    width = int(np.prod(local.shape[1:])) if local.ndim > 1 else 1
    maxrows = shard_range(total, world, 0)[1] - shard_range(total, world, 0)[0]
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros((maxrows, width), dtype=torch.float64, device=dev)
    buf[: hi - lo] = torch.as_tensor(local.reshape(hi - lo, width), dtype=torch.float64, device=dev)
    parts = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    if backend == "nccl":
        parts_all = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts_all, buf, group=group)
        parts = parts_all if rank == 0 else None
    else:
        dist.gather(buf, parts, dst=0, group=group)
    if rank != 0:
        return None
    rows = []
    for r in range(world):
        a, b = shard_range(total, world, r)
        rows.append(parts[r][: b - a].cpu().numpy())
    out = np.concatenate(rows, axis=0)
    return out.reshape((total,) + local.shape[1:]).astype(local.dtype)
