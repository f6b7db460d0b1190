"""Multi-GPU plumbing (north_star: "sharding independent scans in a batch, and
output-voxel ranges of very large scenes ... with NCCL over NVLink only to gather sharded
outputs").

Two splits, neither of which communicates a kernel map:

1. independent scans (``assign_scans``): LPT by voxel count, each rank runs whole scans;
2. one large scene, one layer (``range_shard_plan`` / ``shard_conv`` /
   ``sharded_conv_forward``): rank r owns an equal-count range of the sorted output keys
   and builds its map against the ONE contiguous halo range of input keys its outputs
   can reach (spc_shard_ranges, P:287-290 / P:341), then computes its rows; one
   variable-size all-gather assembles the output in canonical order;
3. one large scene, a layer STACK (``ShardedStack``): the features stay
   distributed by output range between layers; before each layer every rank fetches the
   rows of its input halo that other ranks own (``halo_plan`` / ``exchange_rows``: one
   batch of NCCL send/recv per layer with the ranks whose ranges overlap -- for
   submanifold layers the x-neighbours), so only the final output is gathered.

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



# ---------------------------------------------------------------------------------------
# 3. layer stacks over one scene: per-layer halo exchange
# ---------------------------------------------------------------------------------------

def _overlap(a, b):
    lo, hi = max(a[0], b[0]), min(a[1], b[1])
    return (lo, hi) if lo < hi else None


def halo_plan(own_ranges, need_ranges, rank: int):
    """Host logic of one exchange.  Rank r holds the global rows own_ranges[r] of a
    row-distributed array and needs the contiguous rows need_ranges[r].  Returns
    (sends, recvs, local): sends = [(peer, lo, hi)] rows of this rank that peer needs,
    recvs = [(peer, lo, hi)] rows this rank needs that peer owns, local = the rows it
    needs and owns itself (or None); global row indices, peers in ascending order."""
    sends, recvs = [], []
    for s in range(len(own_ranges)):
        if s == rank:
            continue
        o = _overlap(own_ranges[rank], need_ranges[s])
        if o:
            sends.append((s, o[0], o[1]))
        o = _overlap(own_ranges[s], need_ranges[rank])
        if o:
            recvs.append((s, o[0], o[1]))
    return sends, recvs, _overlap(own_ranges[rank], need_ranges[rank])


def _check_cover(own_ranges, need_ranges, rank):
    """Every needed row is owned by some rank (the ownership ranges tile [0, n))."""
    lo, hi = need_ranges[rank]
    cov = sorted((max(a, lo), min(b, hi)) for a, b in own_ranges if min(b, hi) > max(a, lo))
    at = lo
    for a, b in cov:
        if a > at:
            break
        at = max(at, b)
    if at < hi:
        raise ValueError(f"rows [{at}, {hi}) of rank {rank}'s halo are owned by no rank")


def exchange_rows(owned: torch.Tensor, own_ranges, need_ranges, group=None) -> torch.Tensor:
    """[collective] Rank r passes its owned rows (global rows own_ranges[r]) and receives
    the rows need_ranges[r] as one contiguous tensor: its own overlap is copied, the rest
    arrives by point-to-point send/recv (one batch per call; NCCL over NVLink on GPUs)."""
    rank = dist.get_rank(group)
    _check_cover(own_ranges, need_ranges, rank)
    sends, recvs, local = halo_plan(own_ranges, need_ranges, rank)
    lo_own = own_ranges[rank][0]
    lo_need, hi_need = need_ranges[rank]
    out = torch.empty((hi_need - lo_need,) + tuple(owned.shape[1:]), dtype=owned.dtype, device=owned.device)
    if local:
        out[local[0] - lo_need:local[1] - lo_need] = owned[local[0] - lo_own:local[1] - lo_own]
    ops = []
    for s, lo, hi in sends:
        ops.append(dist.P2POp(dist.isend, owned[lo - lo_own:hi - lo_own].contiguous(), s, group=group))
    bufs = []
    for s, lo, hi in recvs:
        b = torch.empty((hi - lo,) + tuple(owned.shape[1:]), dtype=owned.dtype, device=owned.device)
        bufs.append((lo, b))
        ops.append(dist.P2POp(dist.irecv, b, s, group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for lo, b in bufs:
        out[lo - lo_need:lo - lo_need + b.shape[0]] = b
    return out


def exchange_rows_emulated(owned_list, own_ranges, need_ranges):
    """The same exchange for R ranks emulated in ONE process (single-GPU tests): the
    copies halo_plan prescribes, with no collective (ranks never wait on each other)."""
    outs = []
    for r in range(len(owned_list)):
        _check_cover(own_ranges, need_ranges, r)
        _, recvs, local = halo_plan(own_ranges, need_ranges, r)
        lo_need, hi_need = need_ranges[r]
        o = owned_list[r]
        out = torch.empty((hi_need - lo_need,) + tuple(o.shape[1:]), dtype=o.dtype, device=o.device)
        parts = ([(r, local[0], local[1])] if local else []) + recvs
        for s, lo, hi in parts:
            src_lo = own_ranges[s][0]
            out[lo - lo_need:hi - lo_need] = owned_list[s][lo - src_lo:hi - src_lo]
        outs.append(out)
    return outs


class ShardedStack:
    """A stack of SpC layers over one scene sharded by output ranges.

    ``layers``: list of dicts with keys in_keys, out_keys (the level key arrays of the
    layer, identical on every rank), geom, t, flags, weight (prepared), c_in, c_out and
    optionally residual_from (index of an earlier layer whose output -- same level, hence
    the same ownership ranges -- is added) and epilogue kwargs (scale, shift, relu).
    Maps are built once per layer on this rank's (halo, range) and reused by every
    forward; only the features move (one halo exchange per layer)."""

    def __init__(self, layers, spec, world: int, rank: int, stream=None):
        import paper_2511_20834_b200 as spc
        self.layers, self.world, self.rank = layers, world, rank
        self.plans, self.maps = [], []
        for L in layers:
            plan = range_shard_plan(L["in_keys"], L["out_keys"], spec, L["geom"], world, stream=stream)
            self.plans.append(plan)
            out_lo, out_hi, in_lo, in_hi = plan[rank]
            flags = int(L.get("flags", 0)) & ~spc.SPC_KMAP_HALVE_SYMMETRIC
            self.maps.append(spc.spc_build_kmap(L["in_keys"][in_lo:in_hi], L["out_keys"][out_lo:out_hi], spec,
                                                L["geom"], L.get("t", -1), flags, stream=stream))

    def own_ranges(self, i: int):
        return [(p[0], p[1]) for p in self.plans[i]]

    def need_ranges(self, i: int):
        return [(p[2], p[3]) for p in self.plans[i]]

    def layer_local(self, i: int, x_halo: torch.Tensor, residual=None, out_dtype=None, stream=None):
        """This rank's rows of layer i from its gathered input halo."""
        import paper_2511_20834_b200 as spc
        L = self.layers[i]
        return spc.spc_conv_forward(self.maps[i], x_halo, L["weight"], L["c_in"], L["c_out"], out_dtype=out_dtype,
                                    residual=residual, stream=stream, scale=L.get("scale"), shift=L.get("shift"),
                                    relu=bool(L.get("relu", False)))

    def forward(self, x_owned: torch.Tensor, x_own_ranges, group=None, out_dtype=None, stream=None):
        """[collective] x_owned: this rank's rows x_own_ranges[rank] of the first layer's
        input.  Returns this rank's rows of the last layer (ranges own_ranges(-1))."""
        outs = []
        own, cur = x_own_ranges, x_owned
        for i in range(len(self.layers)):
            halo = exchange_rows(cur, own, self.need_ranges(i), group=group)
            rf = self.layers[i].get("residual_from")
            cur = self.layer_local(i, halo, residual=outs[rf] if rf is not None else None, out_dtype=out_dtype,
                                   stream=stream)
            outs.append(cur)
            own = self.own_ranges(i)
        return cur


def emulated_stack_forward(stacks, x_owned_list, x_own_ranges, out_dtype=None, stream=None):
    """ShardedStack.forward for R ranks emulated in one process (one ShardedStack per
    rank, exchange_rows_emulated instead of send/recv): the single-GPU test path."""
    outs = []
    own, cur = x_own_ranges, list(x_owned_list)
    for i in range(len(stacks[0].layers)):
        halos = exchange_rows_emulated(cur, own, stacks[0].need_ranges(i))
        rf = stacks[0].layers[i].get("residual_from")
        cur = [st.layer_local(i, halos[r], residual=outs[rf][r] if rf is not None else None, out_dtype=out_dtype,
                              stream=stream) for r, st in enumerate(stacks)]
        outs.append(cur)
        own = stacks[0].own_ranges(i)
    return cur
