"""Output-range sharding of one scene, emulated on one GPU: for R in
{2, 3, 4} ranks, every rank's map (outputs [out_lo, out_hi) against the input halo
[in_lo, in_hi) from spc_shard_ranges) with its indices shifted back is exactly its slice
of the single-device map, the shards' maps together ARE the single-device map
(bit-exact), and the concatenated shard features match the oracle's Eq. (2)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc
from paper_2511_20834_b200.distributed import range_shard_plan, shard_conv, shard_out_ranges

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _keys(c, spec):
    return torch.from_numpy(oracle.pack(c, spec.astuple())[0].view(np.int64)).to(DEV)


@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("kind,K,t,flags", [("subm", 3, -1, 8), ("subm", 3, 2, 1), ("subm", 5, 3, 9),
                                            ("strided", 3, -1, 0), ("transposed", 3, 0, 0), ("subm_d2", 3, -1, 0),
                                            # NEXT-3 boxes: the halo extremes of non-centred offsets
                                            ("strided", (2, 2, 2), -1, 0), ("transposed", (2, 2, 2), -1, 0),
                                            ("subm", (4, 2, 3), 2, 0), ("subm", (3, 1, 1), -1, 9)])
def test_range_sharded_map_and_conv(R, kind, K, t, flags):
    coords = synth.make_scan(1, 1)
    spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
    fine = oracle.sort_coords(coords)[0]
    coarse = oracle.downsample(fine, 2)
    d = 2 if kind == "subm_d2" else 1
    if kind.startswith("subm"):
        ic, oc, g = fine, fine, spc.Geom(K, 1, d, 1, 0)
    elif kind == "strided":
        ic, oc, g = fine, coarse, spc.Geom(K, 2, 1, 1, 0)
    else:
        ic, oc, g = coarse, fine, spc.Geom(K, 2, 1, 1, 1)
    ik = _keys(ic, spec)
    ok = ik if oc is ic else _keys(oc, spec)     # one key array for a submanifold layer (halving)
    plan = range_shard_plan(ik, ok, spec, g, R)
    assert [(a, b) for a, b, _, _ in plan] == shard_out_ranges(len(oc), R)
    full = spc.spc_kmap_export(spc.spc_build_kmap(ik, ok, spec, g, t, flags))
    ref = oracle.kmap(ic, oc, K, d, transposed=(kind == "transposed"))
    np.testing.assert_array_equal(full, ref)
    c_in, c_out = 32, 48
    F = synth.make_features(len(ic), c_in, seed=9)
    W = synth.make_weights(g.k_vol(), c_in, c_out, seed=10, nnz_per_out=10)
    Fg = torch.from_numpy(F).to(DEV).bfloat16()
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    parts, outs = [], []
    for b in plan:
        out_lo, out_hi, in_lo, in_hi = b
        assert 0 <= in_lo <= in_hi <= len(ic)
        rows, km = shard_conv(b, ik, ok, spec, g, t, flags, Fg, Wg, c_in, c_out, out_dtype=torch.float32)
        tr = spc.spc_kmap_export(km).astype(np.int64)
        tr[:, 1] += out_lo
        tr[:, 2] += in_lo
        parts.append(tr)
        outs.append(rows.cpu().numpy())
        # a shard's map is exactly the single-device map's rows of its outputs
        sel = (full[:, 1] >= out_lo) & (full[:, 1] < out_hi)
        srt = tr[np.lexsort((tr[:, 2], tr[:, 1], tr[:, 0]))]
        np.testing.assert_array_equal(srt, full[sel])
    allp = np.concatenate(parts)
    allp = allp[np.lexsort((allp[:, 2], allp[:, 1], allp[:, 0]))]
    np.testing.assert_array_equal(allp, full)
    got = np.concatenate(outs).astype(np.float64)
    refF = oracle.conv(ic, oc, K, d, F, W, transposed=(kind == "transposed"))
    assert np.abs(got - refF).max() <= 2e-3 * np.abs(refF).max()


@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_sharded_stack_halo_exchange_emulated(R, dt):
    """a six-layer stack over one scene (3 submanifold with a residual and a
    fused BN/ReLU epilogue, strided down, submanifold, transposed up) sharded over R
    emulated ranks -- features stay distributed by output range and each layer first
    gathers its halo rows (halo_plan copies) -- equals the unsharded stack on the same GPU
    and the fp64 oracle chain."""
    from paper_2511_20834_b200.distributed import ShardedStack, emulated_stack_forward
    coords = synth.make_scan(1, 2)
    spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
    fine = oracle.sort_coords(coords)[0]
    coarse = oracle.downsample(fine, 2)
    kf, kc = _keys(fine, spec), _keys(coarse, spec)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    rng = np.random.default_rng(R)
    chans = [(16, 32), (32, 32), (32, 32), (32, 48), (48, 48), (48, 16)]
    geo = [(kf, kf, fine, fine, spc.Geom(3, 1, 1, 1, 0), False)] * 3 + [
        (kf, kc, fine, coarse, spc.Geom(3, 2, 1, 1, 0), False), (kc, kc, coarse, coarse, spc.Geom(3, 1, 1, 2, 0), False),
        (kc, kf, coarse, fine, spc.Geom(3, 2, 1, 1, 1), True)]
    layers, W64 = [], []
    for i, ((ci, co), (ik, ok, _, _, g, _)) in enumerate(zip(chans, geo)):
        W = synth.make_weights(27, ci, co, seed=30 + i, nnz_per_out=6, dtype=dt)
        W64.append(W)
        L = dict(in_keys=ik, out_keys=ok, geom=g, t=2 if i % 2 else -1, flags=8, c_in=ci, c_out=co,
                 weight=spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).to(tdt)))
        if i == 2:
            L.update(residual_from=0, relu=True,
                     scale=torch.full((co,), 0.9, device=DEV), shift=torch.full((co,), 0.05, device=DEV))
        layers.append(L)
    F = synth.make_features(len(fine), 16, seed=40, dtype=dt)
    Fg = torch.from_numpy(F).to(DEV).to(tdt)
    # unsharded stack on the same GPU (one rank)
    one = ShardedStack(layers, spec, 1, 0)
    y1 = emulated_stack_forward([one], [Fg], [(0, len(fine))], out_dtype=tdt)[0]
    stacks = [ShardedStack(layers, spec, R, r) for r in range(R)]
    own0 = shard_out_ranges(len(fine), R)
    yR = emulated_stack_forward(stacks, [Fg[a:b] for a, b in own0], own0, out_dtype=tdt)
    torch.cuda.synchronize()
    got = torch.cat(yR).float().cpu().numpy().astype(np.float64)
    one_np = y1.float().cpu().numpy().astype(np.float64)
    # oracle chain (fp64, intermediates rounded like the GPU's stored dtype)
    x, outs = F.astype(np.float64), []
    for i, (W, (_, _, ic, oc, g, tr)) in enumerate(zip(W64, geo)):
        y = oracle.conv(ic, oc, 3, g.tensor_stride, x, W, transposed=tr)
        if i == 2:
            y = oracle.bn_relu(y * 0.9 + 0.05, residual=outs[0], relu=True)
        y = synth.round_to(y.astype(np.float32), dt).astype(np.float64) if dt == "bf16" else y
        outs.append(y)
        x = y
    m = np.abs(x).max()
    if dt == "f32":
        assert np.abs(got - one_np).max() <= 1e-5 * m and np.abs(got - x).max() <= 1e-4 * m
    else:   # bf16 intermediates: rounding flips between the two accumulation orders compound
        assert np.abs(got - one_np).max() <= 2e-2 * m and np.abs(got - x).max() <= 2e-2 * m
