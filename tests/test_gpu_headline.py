"""GPU parity on the exact code path bench.py times (VERDICT r1 "next round" item 1).

* (a) C2: MinkUNet-42 on the full ~99k-voxel KITTI-shaped scan, maps built with the
  bench's flags (HALVE_SYMMETRIC | DENSITY_ORDER) and the bench's per-map dataflow t
  (profiles/r2_tuned_t_c2.json, tuned on a different scan; plus the untuned hybrid
  default): all 18 distinct kernel maps bit-exact against the oracle, and every one of
  the 49 layers layer-local on >= 2048 sampled output rows within one bf16 ulp of the
  fp64 Eq. (2) reference (reading A18).  At this size the OS part runs
  256-row density-ordered tiles claimed in tile_order (spc_conv.cu decode_tile).
* (b) tile_order: for 128- and 256-row tiles a permutation of the live tiles, in
  non-increasing weight, the weight of a tile = popcount of its ordered tile mask(s).
* (c) C4-style multi-batch keys (8 scans, bits_b = 3): maps bit-exact (batch isolation
  of the z-delta windows) and a sampled full-size convolution.
* (d) dilated (d = 2) convolution, K = 5 strided and K = 5 transposed convolution.
* (e) a forced window-pool overflow (SPC_OPT_KMAP_POOL_KEYS): the global-memory search
  fallback builds the identical map.
* (f) coordinates exactly at the planned headroom limits: maps bit-exact, no flag; one
  step beyond: SPC_FLAG_RANGE.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD

pytestmark = pytest.mark.gpu
DEV = "cuda"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALL = spc.SPC_KMAP_HALVE_SYMMETRIC | spc.SPC_KMAP_DENSITY_ORDER


def _spec_for(coords, max_stride=16, reach=16):
    return spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), int(coords[:, 0].max()) + 1,
                             max_stride, reach)


def _bf16_ulp_excess(got, ref):
    """max over elements of |got - ref| - (one bf16 ulp of ref + fp32 slack); <= 0 passes."""
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
    return float((np.abs(got - ref) - ulp - 1e-5 * np.abs(ref).max()).max())


def _tuned_t():
    p = os.path.join(ROOT, "profiles", "r2_tuned_t_c2.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return {tuple(int(x) for x in k.strip("()").split(",")): int(v) for k, v in d["dataflow_t"].items()}


def _weights(net, i):
    """W [K^3, C_in, C_out] of layer i from the seeded generator (SparseNet's draw order)."""
    g = torch.Generator().manual_seed(20834)
    for j, s in enumerate(net.layers):
        kv = s.map_key[0] ** 3
        a = math.sqrt(3.0 / (min(kv, 10.0) * s.c_in_flops))
        w = (torch.rand(kv, s.c_in, s.c_out, generator=g) * 2 - 1) * a
        if s.c_in != s.c_in_flops:
            w[:, s.c_in_flops:, :] = 0
        if j == i:
            return w.bfloat16().float().numpy().astype(np.float64)
    raise IndexError(i)


def _map_sets(s, lv):
    K, stride, ts, tr = s.map_key
    lf = int(round(math.log2(ts)))
    if stride == 1:
        return lv[lf], lv[lf]
    if tr:
        return lv[lf + 1], lv[lf]
    return lv[lf], lv[lf + 1]


@pytest.fixture(scope="module")
def c2_scan():
    coords = synth.make_scan(2, 0)
    c0 = oracle.sort_coords(coords)[0]
    lv = [c0] + [oracle.downsample(c0, 2 ** m) for m in range(1, 5)]
    return coords, lv


@pytest.mark.slow
@pytest.mark.parametrize("t_source", ["tuned", "hybrid_default"])
def test_c2_headline_path_all_layers(c2_scan, t_source):
    coords, lv = c2_scan
    n = coords.shape[0]
    spec = _spec_for(coords)
    t = _tuned_t() if t_source == "tuned" else None
    if t_source == "tuned" and t is None:
        pytest.skip("profiles/r2_tuned_t_c2.json not committed")
    net = SparseNet(n, spec, device=DEV, t_override=t)                 # HALVE | DENSITY_ORDER (bench flags)
    feats = torch.zeros(n, C_IN_PAD, dtype=torch.bfloat16, device=DEV)
    feats[:, :4] = torch.from_numpy(synth.make_features(n, 4, seed=synth.scan_seed(2, 0) + 1)).to(DEV).bfloat16()
    net.forward(torch.from_numpy(coords).to(DEV), feats)
    torch.cuda.synchronize()
    assert int(net.status.item()) == 0
    assert net.level_n.cpu().tolist() == [len(x) for x in lv]
    # ---- every distinct map, bit-exact; the level-0 OS part really is 256-row ordered tiles
    for mk, km in net.maps.items():
        s = next(x for x in net.layers if x.map_key == mk)
        inp, out = _map_sets(s, lv)
        K, stride, ts, tr = mk
        ref = oracle.kmap(inp, out, K, ts, transposed=bool(tr))
        np.testing.assert_array_equal(spc.spc_kmap_export(km), ref, err_msg=str(mk))
    km0 = net.maps[(3, 1, 1, 0)]
    if km0.k_dense >= 2:
        assert km0.c.os_rows and (len(lv[0]) + 255) // 256 >= 2 * 148      # device picks 256-row tiles
    # ---- every layer, layer-local, on sampled rows (the GPU's own input to that layer)
    rng = np.random.default_rng(7)
    worst = {}
    for i, s in enumerate(net.layers):
        inp, out = _map_sets(s, lv)
        src = net.bufs[s.src][: len(inp), s.src_col:s.src_col + s.c_in].float().cpu().numpy().astype(np.float64)
        res = None
        if s.residual is not None:
            rb, rc = s.residual
            res = net.bufs[rb][: len(out), rc:rc + s.c_out].float().cpu().numpy().astype(np.float64)
        net.conv(i)
        torch.cuda.synchronize()
        got = net.bufs[s.dst][: len(out), s.dst_col:s.dst_col + s.c_out].float().cpu().numpy().astype(np.float64)
        rows = rng.choice(len(out), min(2048, len(out)), replace=False)
        K, stride, ts, tr = s.map_key
        ref = oracle.conv_rows(inp, out, rows, K, ts, src, _weights(net, i), transposed=bool(tr))
        if res is not None:
            ref = ref + res[rows]
        worst[s.name] = _bf16_ulp_excess(got[rows], ref)
    bad = {k: v for k, v in worst.items() if v > 0}
    assert not bad, bad
    assert len(worst) == 49


def test_tile_order_is_a_weight_sorted_permutation(c2_scan):
    """(b): both halves of tile_order of a density-ordered map."""
    coords, lv = c2_scan
    spec = _spec_for(coords)
    keys = torch.from_numpy(oracle.pack(lv[0], spec.astuple())[0].view(np.int64)).to(DEV)
    for t in (-1, 2):
        km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), t, ALL)
        o128, o256, w128, w256 = [x.cpu().numpy() for x in km.tile_order()]
        _, _, masks = km.density_order()
        m = masks.cpu().numpy().view(np.uint32)
        n = len(lv[0])
        nt128, nt256 = (n + 127) // 128, (n + 255) // 256
        pop = np.array([sum(bin(int(w)).count("1") for w in row) for row in m[:nt128]])
        m256 = np.zeros((nt256, m.shape[1]), np.uint32)
        for tt in range(nt256):
            m256[tt] = m[2 * tt] | (m[2 * tt + 1] if 2 * tt + 1 < nt128 else 0)
        pop256 = np.array([sum(bin(int(w)).count("1") for w in row) for row in m256])
        for order, w, p, nt in ((o128, w128, pop, nt128), (o256, w256, pop256, nt256)):
            assert sorted(order[:nt].tolist()) == list(range(nt))               # a permutation
            np.testing.assert_array_equal(w[:nt], p[order[:nt]])                 # weights of those tiles
            assert (np.diff(w[:nt]) <= 0).all()                                  # heaviest first


@pytest.mark.slow
def test_c4_multibatch_maps_and_sampled_conv():
    """(c): 8 Waymo-shaped scans in one key space (bits_b = 3): the z-delta windows never
    match across scans (batch isolation); a full-size sampled convolution."""
    scans = [synth.make_scan(4, i) for i in range(8)]
    parts = []
    for b, c in enumerate(scans):
        c = c.copy()
        c[:, 0] = b
        parts.append(c)
    coords = np.concatenate(parts)
    spec = _spec_for(coords)
    assert spec.bits_b == 3
    c_t = torch.from_numpy(coords).to(DEV)
    keys, perm, status = spc.spc_pack_sort(c_t, spec)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    c0 = oracle.sort_coords(coords)[0]
    c1 = oracle.downsample(c0, 2)
    lk, ln = spc.spc_downsample(keys, spec, [1])
    n1 = int(ln[0].item())
    assert n1 == len(c1)
    coarse = lk[0, :n1]
    for g, ik, ok, ic, oc, t, fl in ((spc.Geom(3, 1, 1, 1, 0), keys, keys, c0, c0, -1, ALL),
                                     (spc.Geom(3, 1, 1, 1, 0), keys, keys, c0, c0, 2, spc.SPC_KMAP_HALVE_SYMMETRIC),
                                     (spc.Geom(3, 2, 1, 1, 0), keys, coarse, c0, c1, -1, ALL),
                                     (spc.Geom(3, 2, 1, 1, 1), coarse, keys, c1, c0, 0, 0)):
        km = spc.spc_build_kmap(ik, ok, spec, g, t, fl)
        ref = oracle.kmap(ic, oc, 3, 1, transposed=bool(g.transposed))
        got = spc.spc_kmap_export(km)
        np.testing.assert_array_equal(got, ref, err_msg=repr(g))
        # no triple joins two scans
        assert (oc[got[:, 1], 0] == ic[got[:, 2], 0]).all()
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), -1, ALL)
    F = synth.make_features(len(c0), 64, seed=11)
    W = synth.make_weights(27, 64, 64, seed=12, nnz_per_out=10)
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(),
                               spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16()), 64, 64,
                               out_dtype=torch.float32)
    rows = np.random.default_rng(1).choice(len(c0), 4096, replace=False)
    ref = oracle.conv_rows(c0, c0, rows, 3, 1, F, W)
    got = out.cpu().numpy()[rows].astype(np.float64)
    assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max()


def _levels(coords, spec, strides):
    c = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.int32)).to(DEV)
    keys, _, status = spc.spc_pack_sort(c, spec)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    out = {1: (keys, oracle.sort_coords(coords)[0])}
    for s in strides:
        cs = oracle.downsample(coords, s)
        out[s] = (torch.from_numpy(oracle.pack(cs, spec.astuple())[0].view(np.int64)).to(DEV), cs)
    return out


@pytest.mark.parametrize("K,d,kind,t,flags,c_in,c_out", [
    (3, 2, "subm", -1, 0, 32, 32), (3, 2, "subm", 2, 1, 64, 64), (3, 2, "subm", 0, 9, 32, 48),
    (5, 1, "strided", -1, 0, 32, 32), (5, 1, "strided", 3, 8, 32, 64), (5, 1, "strided", 0, 0, 16, 32),
    (5, 1, "transposed", -1, 0, 32, 32), (5, 1, "transposed", 3, 8, 64, 32), (5, 1, "transposed", 0, 0, 32, 16),
    (3, 2, "strided", 2, 8, 32, 32),
])
def test_conv_dilated_and_k5_strided_transposed(K, d, kind, t, flags, c_in, c_out):
    """(d): Eq. (2) with offsets delta * d (reading A11) and K = 5 down / up layers."""
    coords = synth.make_scan(1, 0)[:6000]
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [2])
    fk, fc = lv[1]
    ck, cc = lv[2]
    if kind == "subm":
        ik, ic, ok, oc, g = fk, fc, fk, fc, spc.Geom(K, 1, d, 1, 0)
    elif kind == "strided":
        ik, ic, ok, oc, g = fk, fc, ck, cc, spc.Geom(K, 2, d, 1, 0)
    else:
        ik, ic, ok, oc, g = ck, cc, fk, fc, spc.Geom(K, 2, d, 1, 1)
    km = spc.spc_build_kmap(ik, ok, spec, g, t, flags)
    np.testing.assert_array_equal(spc.spc_kmap_export(km), oracle.kmap(ic, oc, K, d, transposed=(kind == "transposed")))
    F = synth.make_features(len(ic), c_in, seed=c_in + K)
    W = synth.make_weights(K ** 3, c_in, c_out, seed=c_out + K, nnz_per_out=10)
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(),
                               spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16()), c_in, c_out,
                               out_dtype=torch.float32)
    torch.cuda.synchronize()
    # oracle: spacing = d for a dilated layer at tensor stride 1 (Delta(K, s_p) * d)
    ref = oracle.conv(ic, oc, K, d, F, W, transposed=(kind == "transposed"))
    got = out.cpu().numpy().astype(np.float64)
    assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max()


@pytest.mark.parametrize("pool_keys", [0, 64, 300])
def test_window_pool_overflow_fallback(pool_keys):
    """(e): groups whose windows do not fit the (shrunk) shared pool search global memory;
    the map is identical (and the search-count law still holds)."""
    coords = synth.make_scan(1, 1)
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [2])
    fk, fc = lv[1]
    ck, cc = lv[2]
    try:
        spc.spc_set_option(spc.SPC_OPT_KMAP_POOL_KEYS, pool_keys)
        for g, ik, ok, ic, oc, t, fl in ((spc.Geom(3, 1, 1, 1, 0), fk, fk, fc, fc, -1, spc.SPC_KMAP_COUNT_SEARCHES),
                                         (spc.Geom(5, 1, 1, 1, 0), fk, fk, fc, fc, 3, 1 | 8),
                                         (spc.Geom(3, 2, 1, 1, 0), fk, ck, fc, cc, 2, 0),
                                         (spc.Geom(3, 2, 1, 1, 1), ck, fk, cc, fc, -1, 8)):
            km = spc.spc_build_kmap(ik, ok, spec, g, t, fl)
            ref = oracle.kmap(ic, oc, g.kernel_size, 1, transposed=bool(g.transposed))
            np.testing.assert_array_equal(spc.spc_kmap_export(km), ref, err_msg=repr(g))
            if fl & spc.SPC_KMAP_COUNT_SEARCHES:
                assert km.search_stats().cpu().numpy()[0] == len(oc) * 9        # P:297 |V_q| K^2
    finally:
        spc.spc_set_option(spc.SPC_OPT_KMAP_POOL_KEYS, -1)


def test_coordinates_at_the_planned_headroom_limits():
    """(f): a cloud whose extreme coordinates sit exactly at the limits spc_plan_pack
    planned for (reach 2, out_stride 4): pack flags nothing, downsampling and K=5 /
    dilated / strided maps are bit-exact; one coordinate one step further is flagged."""
    rng = np.random.default_rng(3)
    reach, s_max = 2, 4
    # z field of 6 bits: -32 + (s-1) + reach = -27 .. 31 - reach = 29
    lo, hi = np.array([-60, -40, -27]), np.array([61, 40, 29])
    spec = spc.spc_plan_pack(lo, hi, 1, s_max, reach)
    B = (spec.bits_x, spec.bits_y, spec.bits_z)
    for a in range(3):   # the plan is tight: the extremes touch the headroom limit of some field
        assert lo[a] >= -(1 << (B[a] - 1)) + (s_max - 1) + reach and hi[a] <= (1 << (B[a] - 1)) - 1 - reach
    assert lo[2] == -(1 << (B[2] - 1)) + (s_max - 1) + reach and hi[2] == (1 << (B[2] - 1)) - 1 - reach
    pts = set()
    # dense clusters around every corner of the box + random interior points
    for cx in (lo[0], hi[0]):
        for cy in (lo[1], hi[1]):
            for cz in (lo[2], hi[2]):
                for _ in range(60):
                    p = (cx + rng.integers(-2, 3), cy + rng.integers(-2, 3), cz + rng.integers(-2, 3))
                    pts.add(tuple(int(np.clip(v, l, h)) for v, l, h in zip(p, lo, hi)))
    for _ in range(3000):
        pts.add(tuple(int(rng.integers(l, h + 1)) for l, h in zip(lo, hi)))
    coords = np.array([(0,) + p for p in sorted(pts)], np.int32)
    coords = coords[rng.permutation(len(coords))]
    lv = _levels(coords, spec, [2, 4])
    fk, fc = lv[1]
    lk, ln = spc.spc_downsample(fk, spec, [1, 2])
    for l, s in enumerate((2, 4)):
        n_l = int(ln[l].item())
        np.testing.assert_array_equal(lk[l, :n_l].cpu().numpy(), lv[s][0].cpu().numpy())
    for g, ik, ok, ic, oc, K, sp, tr in (
            (spc.Geom(5, 1, 1, 1, 0), fk, fk, fc, fc, 5, 1, False),
            (spc.Geom(3, 1, 2, 1, 0), fk, fk, fc, fc, 3, 2, False),
            (spc.Geom(3, 1, 1, 2, 0), lv[2][0], lv[2][0], lv[2][1], lv[2][1], 3, 2, False),
            (spc.Geom(3, 2, 1, 2, 0), lv[2][0], lv[4][0], lv[2][1], lv[4][1], 3, 2, False),
            (spc.Geom(3, 2, 1, 2, 1), lv[4][0], lv[2][0], lv[4][1], lv[2][1], 3, 2, True)):
        km = spc.spc_build_kmap(ik, ok, spec, g, -1, 0)
        np.testing.assert_array_equal(spc.spc_kmap_export(km), oracle.kmap(ic, oc, K, sp, transposed=tr),
                                      err_msg=repr(g))
    with pytest.raises(spc.SpcError):      # reach 3 > planned 2
        spc.spc_build_kmap(fk, fk, spec, spc.Geom(3, 1, 3, 1, 0), -1, 0)
    for axis, v in ((3, lo[2] - 1), (3, hi[2] + 1), (1, lo[0] - 200)):
        bad = coords.copy()
        bad[5, axis] = v
        _, _, status = spc.spc_pack_sort(torch.from_numpy(bad).to(DEV), spec)
        torch.cuda.synchronize()
        assert int(status.item()) & spc.SPC_FLAG_RANGE, (axis, v)


def test_forced_256_row_tiles_small_input():
    """the 256-row density-ordered OS path (tile_order's second half, os_rows
    scatter) in the fast suite, forced on a small input."""
    coords = synth.make_scan(1, 0)[:7000]
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [])
    fk, fc = lv[1]
    try:
        spc.spc_set_option(spc.SPC_OPT_CONV_TILE_ROWS, 256)
        for t, fl, ci, co in ((-1, ALL, 32, 32), (2, ALL, 64, 96), (-1, ALL, 128, 64), (0, 1, 32, 32)):
            km = spc.spc_build_kmap(fk, fk, spec, spc.Geom(3, 1, 1, 1, 0), t, fl)
            F = synth.make_features(len(fc), ci, seed=ci)
            W = synth.make_weights(27, ci, co, seed=co, nnz_per_out=10)
            out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(),
                                       spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16()), ci, co,
                                       out_dtype=torch.float32)
            ref = oracle.conv(fc, fc, 3, 1, F, W)
            got = out.cpu().numpy().astype(np.float64)
            assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max(), (t, ci, co)
    finally:
        spc.spc_set_option(spc.SPC_OPT_CONV_TILE_ROWS, -1)


def test_variable_scan_size_same_buffers():
    """SparseNet runs a smaller scan on the buffers of its capacity (device live count):
    the result equals a net built for exactly that scan."""
    coords = synth.make_scan(1, 0)
    n_small = coords.shape[0] - 3001
    small = coords[:n_small]
    spec = _spec_for(coords)
    big = SparseNet(coords.shape[0], spec, device=DEV)
    exact = SparseNet(n_small, spec, device=DEV)
    f = torch.zeros(n_small, C_IN_PAD, dtype=torch.bfloat16, device=DEV)
    f[:, :4] = torch.from_numpy(synth.make_features(n_small, 4, seed=5)).to(DEV).bfloat16()
    c = torch.from_numpy(small).to(DEV)
    o1 = big.forward(c, f)[:n_small].float()
    o2 = exact.forward(c, f)[:n_small].float()
    torch.cuda.synchronize()
    assert int(big.status.item()) == 0
    assert big.level_n.cpu().tolist() == exact.level_n.cpu().tolist()
    # same maps and same kernels; WS atomics may reorder fp32 sums (last bits)
    torch.testing.assert_close(o1, o2, rtol=2e-2, atol=2e-2 * float(o2.abs().max()))
