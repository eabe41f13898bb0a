"""Env-sharded multi-GPU plumbing (one process per GPU, torch.distributed).

Environments are independent, so a step has no data-path collective
(SURVEY.md §8(e)): each rank owns a contiguous env slice and its own device
handle. The only collectives are off the step path: the max-over-ranks of
timings and an optional all-gather of per-env rollout statistics (COM,
contacts, finite flags) over NVLink/NVSwitch (NCCL) or gloo on CPU.
"""
from __future__ import annotations

import numpy as np


def env_slice(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [env0, env0+n) of rank among world (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    env0 = rank * base + min(rank, extra)
    return env0, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_env_stats(local: np.ndarray, n_total: int, device=None) -> np.ndarray:
    """All-gather a per-env [n_local, k] float64 array into [n_total, k] in
    rank order (pads to the largest slice for the collective)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return np.asarray(local)
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [env_slice(n_total, world, r)[1] for r in range(world)]
    k = local.shape[1]
    buf = np.zeros((max(sizes), k))
    buf[:local.shape[0]] = local
    t = torch.from_numpy(buf).to(device if device is not None else "cpu")
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    return np.concatenate([o.cpu().numpy()[:sizes[r]] for r, o in enumerate(outs)], axis=0)
