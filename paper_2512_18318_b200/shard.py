"""Multi-GPU host logic of the path (SURVEY.md §8 e): streams are independent,
so stream s is owned by GPU s mod G for its whole life (segmenter state,
mel, generator batches), there is no data-path collective, and the only
cross-rank traffic is the benchmark's bookkeeping: a barrier, the step time
max-reduced over ranks, and the paced latencies gathered to rank 0.

Works with any torch.distributed backend (NCCL on the GPU box, gloo in the
CPU tests); `dist=None` means a single process."""
from __future__ import annotations

import numpy as np


def streams_for_rank(n_total: int, rank: int, world: int) -> list[int]:
    """Global stream ids owned by `rank` out of n_total streams: s mod world
    == rank (strong scaling: the job's stream count is fixed, each of the
    `world` GPUs owns ~n_total / world of them)."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError("streams_for_rank: bad rank/world/count")
    return [s for s in range(n_total) if s % world == rank]


def max_over_ranks(x: float, dist=None, device=None) -> float:
    """Step time of the slowest rank (the job finishes when it does)."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, dist=None, device=None) -> float:
    """Work done by all ranks (e.g. frames rendered: ranks own different streams)."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_arrays(arrays: list[np.ndarray], dist=None, world: int = 1) -> list[np.ndarray]:
    """Concatenate per-rank 1-D arrays (e.g. per-segment latencies) over all
    ranks, rank order; every rank receives the result."""
    if dist is None:
        return [np.asarray(a, np.float64) for a in arrays]
    got = [None] * world
    dist.all_gather_object(got, [np.asarray(a, np.float64).tolist() for a in arrays])
    return [np.array(sum((g[i] for g in got), []), np.float64) for i in range(len(arrays))]
