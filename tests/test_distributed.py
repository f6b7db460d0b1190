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


# ---------------------------------------------------------------------------------------
# layer stacks over one scene, per-layer halo exchange
# ---------------------------------------------------------------------------------------

from paper_2511_20834_b200.distributed import ShardedStack, exchange_rows, halo_plan, shard_out_ranges  # noqa: E402


def test_halo_plan_covers_exactly_once():
    import random
    rnd = random.Random(3)
    for _ in range(200):
        world = rnd.randint(1, 6)
        n = rnd.randint(world, 60)
        cuts = sorted(rnd.sample(range(1, n), world - 1)) if world > 1 else []
        own = list(zip([0] + cuts, cuts + [n]))
        need = []
        for _r in range(world):
            a = rnd.randint(0, n - 1)
            need.append((a, rnd.randint(a + 1, n)))
        plans = [halo_plan(own, need, r) for r in range(world)]
        for r in range(world):
            sends, recvs, local = plans[r]
            got = sorted([(lo, hi) for _, lo, hi in recvs] + ([local] if local else []))
            at = need[r][0]
            for lo, hi in got:
                assert lo == at          # contiguous, no overlap, no gap
                at = hi
            assert at == need[r][1]
            for s, lo, hi in recvs:      # every receive is the peer's matching send
                assert (r, lo, hi) in plans[s][0]
            for s, lo, hi in sends:
                assert own[r][0] <= lo < hi <= own[r][1] and need[s][0] <= lo < hi <= need[s][1]


def _exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 50
        A = torch.arange(n * 3, dtype=torch.float32).view(n, 3)
        own = [(0, 17), (17, 31), (31, 50)][:world] if world == 3 else shard_out_ranges(n, world)
        need = [(0, 40), (5, 50), (12, 33)][:world]
        got = exchange_rows(A[own[rank][0]:own[rank][1]].clone(), own, need)
        ok = torch.equal(got, A[need[rank][0]:need[rank][1]])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(res, key=lambda x: x[0])


def test_exchange_rows_gloo_world3():
    res = _spawn(_exchange_worker, 3)
    assert [r[0] for r in res] == [0, 1, 2] and all(r[1] for r in res)


class _OracleStack(ShardedStack):
    """ShardedStack whose plans and rank-local compute come from the CPU oracle (test
    infrastructure standing in for spc_shard_ranges / spc_conv_forward, which need a GPU):
    the exchange, ownership and residual bookkeeping under test are the product's."""

    def __init__(self, layers, world, rank):
        import numpy as np
        import oracle
        self.layers, self.world, self.rank = layers, world, rank
        self.plans = []
        for L in layers:
            trip = oracle.kmap(L["in_c"], L["out_c"], L["K"], 1, transposed=L.get("transposed", False))
            plan = []
            for lo, hi in shard_out_ranges(len(L["out_c"]), world):
                sel = trip[(trip[:, 1] >= lo) & (trip[:, 1] < hi)][:, 2]
                a, b = (int(sel.min()), int(sel.max()) + 1) if len(sel) else (0, 0)
                plan.append((lo, hi, a, b))
            self.plans.append(plan)
        self._np = np

    def layer_local(self, i, x_halo, residual=None, out_dtype=None, stream=None):
        import oracle
        L = self.layers[i]
        out_lo, out_hi, in_lo, in_hi = self.plans[i][self.rank]
        y = oracle.conv(L["in_c"][in_lo:in_hi], L["out_c"][out_lo:out_hi], L["K"], 1, x_halo.numpy(), L["W"],
                        transposed=L.get("transposed", False))
        y = torch.from_numpy(y)
        return y + residual if residual is not None else y


def _stack_layers():
    import numpy as np
    import oracle
    import synth
    fine = oracle.sort_coords(synth.make_scan(1, 0)[:1500])[0]
    coarse = oracle.downsample(fine, 2)
    rng = np.random.default_rng(0)
    W = lambda k, a, b: rng.uniform(-0.3, 0.3, (k, a, b))
    layers = [dict(in_c=fine, out_c=fine, K=3, W=W(27, 4, 6)),
              dict(in_c=fine, out_c=fine, K=3, W=W(27, 6, 6)),
              dict(in_c=fine, out_c=fine, K=3, W=W(27, 6, 6), residual_from=0),
              dict(in_c=fine, out_c=coarse, K=3, W=W(27, 6, 5)),          # strided: level change
              dict(in_c=coarse, out_c=coarse, K=3, W=W(27, 5, 5)),
              dict(in_c=coarse, out_c=fine, K=3, W=W(27, 5, 3), transposed=True)]   # back up
    F = rng.uniform(-1, 1, (len(fine), 4))
    return layers, F


def _stack_ref(layers, F):
    import oracle
    outs, x = [], F
    for L in layers:
        y = oracle.conv(L["in_c"], L["out_c"], L["K"], 1, x, L["W"], transposed=L.get("transposed", False))
        if L.get("residual_from") is not None:
            y = y + outs[L["residual_from"]]
        outs.append(y)
        x = y
    return x


def _stack_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers, F = _stack_layers()
        st = _OracleStack(layers, world, rank)
        own0 = shard_out_ranges(len(F), world)
        x = torch.from_numpy(F[own0[rank][0]:own0[rank][1]])
        y = st.forward(x, own0)
        full = torch.cat(gather_rows(y))
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_stack_halo_exchange_gloo(world):
    """Six layers (3 submanifold with a residual, strided down, submanifold, transposed up)
    sharded over `world` gloo ranks equal the unsharded stack (fp64 oracle compute)."""
    import numpy as np
    res = _spawn(_stack_worker, world)
    layers, F = _stack_layers()
    ref = _stack_ref(layers, F)
    for _, full in res:
        np.testing.assert_allclose(full, ref, rtol=1e-12, atol=1e-12)
