"""Host logic of the multi-GPU path on CPU: world_size-2 gloo process group."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_20834_b200.distributed import assign_scans, gather_rows, max_over_ranks


def test_assign_scans_lpt_balanced():
    sizes = [207_000, 129_000, 181_000, 150_000, 199_000, 170_000, 160_000, 140_000]
    a = assign_scans(sizes, 8)
    assert sorted(sum(a, [])) == list(range(8)) and all(len(x) == 1 for x in a)
    a2 = assign_scans(sizes, 2)
    loads = [sum(sizes[i] for i in x) for x in a2]
    assert sorted(sum(a2, [])) == list(range(8))
    assert max(loads) - min(loads) <= max(sizes)
    assert assign_scans(sizes, 3) == assign_scans(sizes, 3)   # deterministic


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = 3 + 2 * rank                                   # different row counts per rank
        t = torch.full((rows, 4), float(rank), dtype=torch.float32)
        t[:, 0] = torch.arange(rows, dtype=torch.float32)
        parts = gather_rows(t)
        ok = [p.shape[0] == 3 + 2 * r and bool((p[:, 1:] == r).all()) for r, p in enumerate(parts)]
        m = max_over_ranks(1.5 + rank)
        q.put((rank, all(ok), m))
    finally:
        dist.destroy_process_group()


def test_gather_rows_and_max_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res)
    assert all(abs(r[2] - 2.5) < 1e-12 for r in res)


def _range_worker(rank, world, port, q):
    """Range sharding plumbing on gloo: each rank produces the rows of its equal-count
    output range; the variable-size gather reassembles the canonical order."""
    from paper_2511_20834_b200.distributed import shard_out_ranges
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1001
        lo, hi = shard_out_ranges(n, world)[rank]
        rows = torch.arange(lo, hi, dtype=torch.float64)[:, None] * torch.tensor([[1.0, -2.0, 0.5]])
        full = torch.cat(gather_rows(rows))
        ref = torch.arange(n, dtype=torch.float64)[:, None] * torch.tensor([[1.0, -2.0, 0.5]])
        q.put((rank, bool(torch.equal(full, ref))))
    finally:
        dist.destroy_process_group()


def test_shard_out_ranges_cover_and_balance():
    from paper_2511_20834_b200.distributed import shard_out_ranges
    for n, w in ((0, 3), (7, 8), (100_000, 8), (98_895, 3)):
        r = shard_out_ranges(n, w)
        assert r[0][0] == 0 and r[-1][1] == n and all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [h - l for l, h in r]
        assert max(sizes) - min(sizes) <= 1


def test_range_shard_gather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_range_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1] and all(r[1] for r in res)
