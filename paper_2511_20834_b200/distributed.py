"""Multi-GPU plumbing (north_star: "sharding independent scans in a batch, and
output-voxel ranges of very large scenes ... with NCCL over NVLink only to gather sharded
outputs").

Two splits, neither of which communicates a kernel map:

1. independent scans (``assign_scans``): LPT by voxel count, each rank runs whole scans;
2. one large scene, one layer (``range_shard_plan`` / ``shard_conv`` /
   ``sharded_conv_forward``): rank r owns an equal-count range of the sorted output keys
   and builds its map against the ONE contiguous halo range of input keys its outputs
   can reach (spc_shard_ranges, P:287-290 / P:341), then computes its rows; one
   variable-size all-gather assembles the output in canonical order.

Works on any torch.distributed backend (NCCL for CUDA tensors, gloo for CPU tensors in
the tests).
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


def shard_out_ranges(n: int, world: int):
    """Equal-count output ranges [r*n/world, (r+1)*n/world) (the split spc_shard_ranges uses)."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def range_shard_plan(in_keys, out_keys, spec, geom, world: int, stream=None):
    """[sync] per-rank (out_lo, out_hi, in_lo, in_hi) of one layer's map (spc_shard_ranges)."""
    import paper_2511_20834_b200 as spc
    b = spc.spc_shard_ranges(in_keys, out_keys, spec, geom, world, stream=stream)
    return [tuple(int(v) for v in row) for row in b.cpu().tolist()]


def shard_conv(bounds, in_keys, out_keys, spec, geom, t, flags, f_in, weight_prepared, c_in: int, c_out: int,
               out_dtype=None, stream=None):
    """Rank-local part of one layer: the map of outputs [out_lo, out_hi) against the input
    halo [in_lo, in_hi) and its features.  Returns (rows [out_hi - out_lo, c_out], map)."""
    import paper_2511_20834_b200 as spc
    out_lo, out_hi, in_lo, in_hi = bounds
    # a shard's input and output index spaces differ: no symmetric halving (it needs one set)
    flags = int(flags) & ~spc.SPC_KMAP_HALVE_SYMMETRIC
    km = spc.spc_build_kmap(in_keys[in_lo:in_hi], out_keys[out_lo:out_hi], spec, geom, t, flags, stream=stream)
    out = spc.spc_conv_forward(km, f_in[in_lo:in_hi], weight_prepared, c_in, c_out, out_dtype=out_dtype,
                               stream=stream)
    return out, km


def sharded_conv_forward(in_keys, out_keys, spec, geom, t, flags, f_in, weight_prepared, c_in: int, c_out: int,
                         out_dtype=None, group=None, stream=None):
    """One layer over a scene too large for one GPU's step budget: every rank computes its
    output range, then one variable-size all-gather (the only collective) returns the whole
    [n_out, c_out] output, in canonical order, on every rank."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    plan = range_shard_plan(in_keys, out_keys, spec, geom, world, stream=stream)
    rows, _ = shard_conv(plan[rank], in_keys, out_keys, spec, geom, t, flags, f_in, weight_prepared, c_in, c_out,
                         out_dtype=out_dtype, stream=stream)
    return torch.cat(gather_rows(rows, group=group))

