"""Multi-GPU plumbing for the scan-sharded path (north_star: "sharding independent scans
in a batch ... with NCCL over NVLink only to gather sharded outputs").

Kernel maps never cross GPUs; the only data-path collective is gathering the per-rank
output features (variable row counts) after the forward passes.  Works on any
torch.distributed backend (NCCL for CUDA tensors, gloo for CPU tensors in tests).
"""
from __future__ import annotations

import heapq

import torch
import torch.distributed as dist


def assign_scans(sizes, world: int):
    """Longest-processing-time assignment of scans (by voxel count) to ranks.
    Returns a list of scan-index lists, one per rank (deterministic)."""
    order = sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))
    heap = [(0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(sizes[i]), r))
    return [sorted(x) for x in out]


def gather_rows(t: torch.Tensor, group=None):
    """All-gather a [rows, ...] tensor whose row count differs per rank.
    Returns the list of per-rank tensors (padded all_gather + trim)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    m = max(ns)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[:k] for b, k in zip(bufs, ns)]


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timing rule: slowest rank defines the step)."""
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
