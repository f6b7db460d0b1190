"""GPU parity: every step of the CUDA hot path (through the C ABI) against the CPU oracle.

Integer work (keys, permutation, downsampled sets, kernel maps) must be bit-exact;
features within north_star's tolerance: max|gpu - ref| <= 2e-3 * max|ref| for f16/bf16
inputs (fp32 output), <= 1e-5 * max|ref| for the fp32 path; bf16/f16-stored outputs are
checked against round(ref) to within one unit in the last place (reading A18).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _spec_for(coords, max_stride=16, reach=16):
    lo = coords[:, 1:].min(0)
    hi = coords[:, 1:].max(0)
    nb = int(coords[:, 0].max()) + 1
    return spc.spc_plan_pack(lo, hi, nb, max_stride, reach)


def _pack_sort(coords, spec):
    c = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.int32)).to(DEV)
    keys, perm, status = spc.spc_pack_sort(c, spec)
    torch.cuda.synchronize()
    return keys, perm, int(status.item())


def _keys_of(coords_sorted, spec):
    k, bad = oracle.pack(coords_sorted, spec.astuple())
    assert bad == 0
    return k.view(np.int64)


# ---------------------------------------------------------------------------------------
# A1 + A2
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["c1", "random_batched", "tiny", "one"])
def test_pack_sort_bit_exact(case):
    if case == "c1":
        coords = synth.make_scan(1, 0)
    elif case == "random_batched":
        coords = synth.random_cloud(50_000, 600, seed=3, n_batch=5)
    elif case == "tiny":
        coords = synth.random_cloud(37, 20, seed=4)
    else:
        coords = np.array([[0, 5, -3, 2]], np.int32)
    spec = _spec_for(coords)
    keys, perm, status = _pack_sort(coords, spec)
    s, p, dups = oracle.sort_coords(coords)
    assert dups == 0 and status == 0
    np.testing.assert_array_equal(keys.cpu().numpy(), _keys_of(s, spec))
    np.testing.assert_array_equal(perm.cpu().numpy(), p)


def test_pack_sort_flags_duplicates_and_range():
    coords = synth.random_cloud(3000, 100, seed=9)
    dup = np.concatenate([coords, coords[:5]])
    spec = _spec_for(coords)
    _, _, status = _pack_sort(dup, spec)
    assert status & spc.SPC_FLAG_DUPLICATE
    bad = coords.copy()
    bad[7, 1] = 1 << (spec.bits_x - 1)          # one past the top of the x field
    _, _, status = _pack_sort(bad, spec)
    assert status & spc.SPC_FLAG_RANGE


def test_gather_rows():
    coords = synth.random_cloud(5000, 200, seed=1)
    spec = _spec_for(coords)
    keys, perm, _ = _pack_sort(coords, spec)
    F = torch.randn(5000, 48, device=DEV).to(torch.bfloat16)
    out = spc.spc_gather_rows(F, perm)
    torch.testing.assert_close(out, F[perm.long()], rtol=0, atol=0)


# ---------------------------------------------------------------------------------------
# A3
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("config", [1, 2])
def test_downsample_levels_bit_exact(config):
    coords = synth.make_scan(config, 0)
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    lv, ln = spc.spc_downsample(keys, spec, [1, 2, 3, 4])
    torch.cuda.synchronize()
    ln = ln.cpu().numpy()
    for l, m in enumerate([1, 2, 3, 4]):
        ref = oracle.downsample(coords, 2 ** m)
        assert ln[l] == len(ref)
        np.testing.assert_array_equal(lv[l, :ln[l]].cpu().numpy(), _keys_of(ref, spec))


@pytest.mark.parametrize("case", ["one_slab", "batched", "tiny", "live_count"])
def test_downsample_segments_edge_cases(case):
    """The segmented downsample sorts each (batch, x >> m) group of rows on its own: a group
    with more distinct keys than the shared hash set holds (one x-slab of 60k voxels: the
    global-memory path), groups split by the batch field, one- and two-voxel inputs, and a live count
    below the capacity (rows past it ignored)."""
    rng = np.random.default_rng(5)
    if case == "one_slab":
        yz = rng.choice(400 * 400, 60000, replace=False)   # level 1: ~34k distinct keys in one run
        coords = np.stack([np.zeros(60000), np.full(60000, 3), yz // 400 - 200, yz % 400 - 200], 1).astype(np.int32)
    elif case == "batched":
        coords = np.concatenate([synth.make_scan(1, 0)[:5000] * np.array([0, 1, 1, 1]) + np.array([b, 0, 0, 0])
                                 for b in range(4)]).astype(np.int32)
    elif case == "tiny":
        coords = np.array([[0, -3, 5, 1], [0, -4, 5, 1]], np.int32)
    else:
        coords = synth.make_scan(2, 0)
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    n_live = len(keys)
    if case == "live_count":   # the first 60000 sorted voxels as a live prefix of the capacity
        n_live = 60000
        c_sorted = oracle.sort_coords(coords)[0][:n_live]
        n_dev = torch.tensor([n_live], dtype=torch.int64, device=DEV)
        lv, ln = spc.spc_downsample(keys, spec, [1, 2, 3, 4], n_dev=n_dev)
    else:
        c_sorted = oracle.sort_coords(coords)[0]
        lv, ln = spc.spc_downsample(keys, spec, [1, 2, 3, 4])
    torch.cuda.synchronize()
    ln = ln.cpu().numpy()
    for l, m in enumerate([1, 2, 3, 4]):
        ref = oracle.downsample(c_sorted, 2 ** m)
        assert ln[l] == len(ref)
        np.testing.assert_array_equal(lv[l, :ln[l]].cpu().numpy(), _keys_of(ref, spec))


# ---------------------------------------------------------------------------------------
# A4-A8 kernel maps
# ---------------------------------------------------------------------------------------

def _levels(coords, spec, strides):
    keys, _, _ = _pack_sort(coords, spec)
    out = {1: (keys, oracle.sort_coords(coords)[0])}
    for s in strides:
        c = oracle.downsample(coords, s)
        k = torch.from_numpy(_keys_of(c, spec)).to(DEV)
        out[s] = (k, c)
    return out


MAP_CASES = [
    # (K, dilation, kind, t, flags)
    (3, 1, "subm", -1, 0), (3, 1, "subm", 0, 0), (3, 1, "subm", 2, 0), (3, 1, "subm", 0, 1), (3, 1, "subm", 2, 1),
    (5, 1, "subm", -1, 0), (5, 1, "subm", 3, 0), (5, 1, "subm", 3, 1), (5, 1, "subm", 0, 1),
    (1, 1, "subm", -1, 0), (3, 2, "subm", 2, 1),
    (3, 1, "strided", -1, 0), (3, 1, "strided", 0, 0), (3, 1, "strided", 2, 0), (5, 1, "strided", 3, 0),
    (3, 1, "transposed", -1, 0), (3, 1, "transposed", 2, 0),
]


@pytest.mark.parametrize("K,d,kind,t,flags", MAP_CASES)
def test_kmap_bit_exact(K, d, kind, t, flags):
    coords = synth.make_scan(1, 1)
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [2])
    fine_k, fine_c = lv[1]
    coarse_k, coarse_c = lv[2]
    if kind == "subm":
        g = spc.Geom(K, 1, d, 1, 0)
        km = spc.spc_build_kmap(fine_k, fine_k, spec, g, t, flags | spc.SPC_KMAP_COUNT_SEARCHES)
        ref = oracle.kmap(fine_c, fine_c, K, d)
        n_out = len(fine_c)
    elif kind == "strided":
        g = spc.Geom(K, 2, d, 1, 0)
        km = spc.spc_build_kmap(fine_k, coarse_k, spec, g, t, flags)
        ref = oracle.kmap(fine_c, coarse_c, K, d)
        n_out = len(coarse_c)
    else:
        g = spc.Geom(K, 2, d, 1, 1)
        km = spc.spc_build_kmap(coarse_k, fine_k, spec, g, t, flags)
        ref = oracle.kmap(coarse_c, fine_c, K, d, transposed=True)
        n_out = len(fine_c)
    got = spc.spc_kmap_export(km)
    np.testing.assert_array_equal(got, ref)
    if kind == "subm":
        st = km.search_stats().cpu().numpy()
        if not (flags & 1):
            assert st[0] == n_out * K * K                              # P:297 |V_q| K^2 searches
            assert st[1] <= n_out * K * K * (K - 1) * d                # <= (K-1)d advances each
        else:
            assert st[0] <= n_out * K * K                              # halving skips groups


@pytest.mark.parametrize("K,d,kind", [(3, 1, "subm"), (5, 1, "subm"), (3, 2, "subm"), (3, 1, "strided"),
                                      (3, 1, "transposed"), (1, 1, "subm")])
def test_kmap_simple_bsearch_ablation(K, d, kind):
    """NEXT-1 ablation: the paper's Simple BSearch mapping builds the same map
    as the oracle with exactly |V_q| K^3 binary searches; it needs an all-OS t."""
    coords = synth.make_scan(1, 1)
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [2])
    fine_k, fine_c = lv[1]
    coarse_k, coarse_c = lv[2]
    fl = spc.SPC_KMAP_SIMPLE_BSEARCH | spc.SPC_KMAP_COUNT_SEARCHES
    if kind == "subm":
        km = spc.spc_build_kmap(fine_k, fine_k, spec, spc.Geom(K, 1, d, 1, 0), -1, fl)
        ref, n_out = oracle.kmap(fine_c, fine_c, K, d), len(fine_c)
    elif kind == "strided":
        km = spc.spc_build_kmap(fine_k, coarse_k, spec, spc.Geom(K, 2, d, 1, 0), -1, fl)
        ref, n_out = oracle.kmap(fine_c, coarse_c, K, d), len(coarse_c)
    else:
        km = spc.spc_build_kmap(coarse_k, fine_k, spec, spc.Geom(K, 2, d, 1, 1), -1, fl)
        ref, n_out = oracle.kmap(coarse_c, fine_c, K, d, transposed=True), len(fine_c)
    np.testing.assert_array_equal(spc.spc_kmap_export(km), ref)
    assert km.search_stats().cpu().numpy()[0] == n_out * K ** 3          # P:257-259 |V_q| K^3 searches
    # the tile mask marks exactly the (128-row tile, offset) chunks with a match
    tab = km.os_table().cpu().numpy().reshape(n_out, -1)
    words = km.tile_mask().cpu().numpy().view(np.uint32)
    for t0 in range(0, n_out, 128):
        any_c = (tab[t0:t0 + 128] >= 0).any(0)
        got = np.array([(words[t0 // 128, c // 32] >> (c % 32)) & 1 for c in range(tab.shape[1])], bool)
        assert np.array_equal(got, any_c)
    with pytest.raises(spc.SpcError):
        spc.spc_build_kmap(fine_k, fine_k, spec, spc.Geom(3, 1, 1, 1, 0), 2, spc.SPC_KMAP_SIMPLE_BSEARCH)


def test_kmap_os_table_exact_and_centre():
    coords = synth.make_scan(1, 0)
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), -1, 0)
    tab = km.os_table().cpu().numpy()
    ref = np.full((len(c), 27), -1, np.int32)
    tr = oracle.kmap(c, c, 3, 1)
    ref[tr[:, 1], tr[:, 0]] = tr[:, 2]
    np.testing.assert_array_equal(tab, ref)
    assert (tab[:, 13] == np.arange(len(c))).all()          # centre maps i -> i


@pytest.mark.parametrize("K,kind,t", [(3, "subm", -1), (3, "subm", 2), (5, "subm", 3), (3, "strided", -1),
                                      (3, "transposed", -1)])
def test_kmap_density_order_exact(K, kind, t):
    """SPC_KMAP_DENSITY_ORDER: os_rows is the STABLE sort of the outputs by the key
    ((16 - popcount(dirs)) << 16) | dirs, dirs bit j set iff the output matches offset k or
    its mirror K^3-1-k (j = rank of the pair min(k, mirror) among the pairs with a dense
    member, the submanifold centre pair skipped, folded mod 16): most directions first,
    then grouped by pattern -- unique, so checked bit-exactly against numpy's stable
    argsort of the oracle map; the ordered table is the canonical one permuted; tile
    masks are the OR of each 128-row tile."""
    coords = synth.make_scan(1, 1)
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [2])
    fine_k, fine_c = lv[1]
    coarse_k, coarse_c = lv[2]
    if kind == "subm":
        g, ik, ok, ic, oc = spc.Geom(K, 1, 1, 1, 0), fine_k, fine_k, fine_c, fine_c
    elif kind == "strided":
        g, ik, ok, ic, oc = spc.Geom(K, 2, 1, 1, 0), fine_k, coarse_k, fine_c, coarse_c
    else:
        g, ik, ok, ic, oc = spc.Geom(K, 2, 1, 1, 1), coarse_k, fine_k, coarse_c, fine_c
    km = spc.spc_build_kmap(ik, ok, spec, g, t, spc.SPC_KMAP_DENSITY_ORDER)
    rows, tab_ord, masks = [x.cpu().numpy() for x in km.density_order()]
    tab = km.os_table().cpu().numpy()
    ref = oracle.kmap(ic, oc, K, 1, transposed=(kind == "transposed"))
    n, kd = tab.shape
    dense = km.dense_k
    col = {k: c for c, k in enumerate(dense)}
    full = np.full((n, kd), -1, np.int64)
    sel = np.isin(ref[:, 0], dense)
    full[ref[sel, 1], [col[k] for k in ref[sel, 0]]] = ref[sel, 2]
    np.testing.assert_array_equal(tab, full)
    kv = K ** 3
    centre = (kv - 1) // 2
    pairs = sorted({min(k, kv - 1 - k) for k in dense if not (kind == "subm" and k == centre)})
    rank = {pr: i % 16 for i, pr in enumerate(pairs)}
    key = np.zeros(n, np.int64)
    for c, k in enumerate(dense):
        pr = min(k, kv - 1 - k)
        if pr in rank:
            key |= (full[:, c] >= 0).astype(np.int64) << rank[pr]
    pop = np.array([bin(int(x)).count("1") for x in key])
    key = ((16 - pop) << 16) | key
    np.testing.assert_array_equal(rows, np.argsort(key, kind="stable"))
    np.testing.assert_array_equal(tab_ord, full[rows])
    pad = (-n) % 128
    hit = np.concatenate([(full[rows] >= 0), np.zeros((pad, kd), bool)]).reshape(-1, 128, kd).any(axis=1)
    words = np.zeros((hit.shape[0], masks.shape[1]), np.int64)
    for c in range(kd):
        words[:, c // 32] |= hit[:, c].astype(np.int64) << (c % 32)
    np.testing.assert_array_equal(masks.view(np.uint32).astype(np.int64), words)


def test_kmap_edge_cases():
    spec = spc.PackSpec(0, 8, 8, 8, 1, 1)
    one = torch.tensor([(128 << 16) | (128 << 8) | 128], dtype=torch.int64, device=DEV)
    km = spc.spc_build_kmap(one, one, spec, spc.Geom(3, 1, 1, 1, 0), -1, 0)
    assert spc.spc_kmap_export(km).tolist() == [[13, 0, 0]]
    empty = torch.empty(0, dtype=torch.int64, device=DEV)
    km = spc.spc_build_kmap(one, empty, spec, spc.Geom(3, 1, 1, 1, 0), -1, 0)
    assert spc.spc_kmap_export(km).shape == (0, 3)
    km = spc.spc_build_kmap(empty, one, spec, spc.Geom(3, 1, 1, 1, 0), 0, 0)
    assert spc.spc_kmap_export(km).shape == (0, 3)
    with pytest.raises(spc.SpcError):
        spc.spc_build_kmap(one, one, spec, spc.Geom(4, 1, 1, 1, 0), -1, 0)


def test_network_kmaps_equal_sequential():
    coords = synth.make_scan(1, 0)
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    geoms = [spc.Geom(3, 1, 1, 1, 0), spc.Geom(3, 2, 1, 1, 0), spc.Geom(3, 1, 1, 2, 0), spc.Geom(3, 2, 1, 2, 0),
             spc.Geom(3, 1, 1, 4, 0), spc.Geom(3, 2, 1, 2, 1), spc.Geom(3, 2, 1, 1, 1), spc.Geom(3, 1, 1, 1, 0)]
    ts = [-1, 0, 2, -1, 0, -1, 2, -1]
    lk, ln, maps = spc.spc_network_kmaps(keys, spec, 4, geoms, ts)
    c = oracle.sort_coords(coords)[0]
    lv = {1: c, 2: oracle.downsample(c, 2), 4: oracle.downsample(c, 4), 8: oracle.downsample(c, 8)}
    assert ln.cpu().tolist() == [len(lv[1]), len(lv[2]), len(lv[4]), len(lv[8])]
    for g, km in zip(geoms, maps):
        fine, coarse = lv[g.tensor_stride], lv[g.tensor_stride * g.stride]
        if g.transposed:
            ref = oracle.kmap(coarse, fine, 3, g.tensor_stride, transposed=True)
        else:
            ref = oracle.kmap(fine, coarse, 3, g.tensor_stride)
        np.testing.assert_array_equal(spc.spc_kmap_export(km), ref)


# ---------------------------------------------------------------------------------------
# A9-A12 features
# ---------------------------------------------------------------------------------------

def _rel_err(got, ref):
    m = np.abs(ref).max()
    return np.abs(got - ref).max() / (m if m > 0 else 1.0)


CONV_CASES = [
    # (K, kind, t, flags, c_in, c_out, dtype)
    (3, "subm", -1, 0, 16, 16, "bf16"), (3, "subm", 0, 1, 32, 32, "bf16"), (3, "subm", 2, 1, 64, 96, "bf16"),
    (3, "subm", 2, 0, 32, 64, "f16"), (5, "subm", 3, 1, 32, 32, "bf16"), (5, "subm", -1, 0, 16, 16, "bf16"),
    (3, "subm", -1, 0, 128, 128, "bf16"), (3, "subm", 0, 1, 256, 256, "bf16"), (1, "subm", -1, 0, 96, 32, "bf16"),
    (3, "strided", -1, 0, 32, 64, "bf16"), (3, "strided", 0, 0, 64, 64, "bf16"),
    (3, "transposed", -1, 0, 64, 32, "bf16"), (3, "transposed", 2, 0, 48, 384, "bf16"),
    (3, "subm", 2, 1, 16, 32, "f32"), (3, "strided", 0, 0, 32, 16, "f32"),
    # density-ordered OS part (SPC_KMAP_DENSITY_ORDER = 8): all-OS, hybrid, strided, transposed, K=5, f32
    (3, "subm", -1, 8, 32, 32, "bf16"), (3, "subm", 2, 9, 64, 96, "bf16"), (3, "strided", -1, 8, 32, 64, "bf16"),
    (3, "transposed", -1, 8, 64, 32, "bf16"), (5, "subm", 3, 9, 32, 32, "bf16"), (3, "subm", -1, 8, 16, 32, "f32"),
]


@pytest.mark.parametrize("K,kind,t,flags,c_in,c_out,dt", CONV_CASES)
def test_conv_forward_matches_eq2(K, kind, t, flags, c_in, c_out, dt):
    coords = synth.make_scan(1, 0)[:6000]
    spec = _spec_for(coords)
    lv = _levels(coords, spec, [2])
    fine_k, fine_c = lv[1]
    coarse_k, coarse_c = lv[2]
    if kind == "subm":
        inp_k, inp_c, out_k, out_c, g = fine_k, fine_c, fine_k, fine_c, spc.Geom(K, 1, 1, 1, 0)
    elif kind == "strided":
        inp_k, inp_c, out_k, out_c, g = fine_k, fine_c, coarse_k, coarse_c, spc.Geom(K, 2, 1, 1, 0)
    else:
        inp_k, inp_c, out_k, out_c, g = coarse_k, coarse_c, fine_k, fine_c, spc.Geom(K, 2, 1, 1, 1)
    km = spc.spc_build_kmap(inp_k, out_k, spec, g, t, flags)
    F = synth.make_features(len(inp_c), c_in, seed=c_in + K, dtype=dt)
    W = synth.make_weights(K ** 3, c_in, c_out, seed=c_out + K, nnz_per_out=10, dtype=dt)
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dt]
    Fg = torch.from_numpy(F).to(DEV).to(tdt)
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).to(tdt))
    out = spc.spc_conv_forward(km, Fg, Wg, c_in, c_out, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle.conv(inp_c, out_c, K, 1, F.astype(np.float64), W.astype(np.float64),
                      transposed=(kind == "transposed"))
    err = _rel_err(out.cpu().numpy().astype(np.float64), ref)
    tol = 1e-5 if dt == "f32" else 2e-3
    assert err <= tol, err


def test_conv_bf16_output_and_residual():
    coords = synth.make_scan(1, 0)[:5000]
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    for t, flags in ((-1, 0), (1, 1)):
        km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), t, flags)
        F = synth.make_features(len(c), 32, seed=1)
        W = synth.make_weights(27, 32, 32, seed=2, nnz_per_out=10)
        R = synth.make_features(len(c), 32, seed=3)
        Fg = torch.from_numpy(F).to(DEV).bfloat16()
        Rg = torch.from_numpy(R).to(DEV).bfloat16()
        Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
        out = spc.spc_conv_forward(km, Fg, Wg, 32, 32, out_dtype=torch.bfloat16, residual=Rg)
        ref = oracle.conv(c, c, 3, 1, F, W) + R.astype(np.float64)
        got = out.float().cpu().numpy().astype(np.float64)
        # one bf16 ulp of the reference value (2^-7 relative to its binade) + fp32 slack
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        assert (np.abs(got - ref) <= ulp + 1e-6 * np.abs(ref).max()).all()


def test_conv_channel_slices():
    """ld_in / ld_out > c: read from and write into column slices (free skip concat)."""
    coords = synth.make_scan(1, 0)[:4000]
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), 2, 1)
    F = synth.make_features(len(c), 64, seed=5)
    W = synth.make_weights(27, 32, 48, seed=6, nnz_per_out=10)
    Fg = torch.from_numpy(F).to(DEV).bfloat16()
    big = torch.zeros(len(c), 96, dtype=torch.float32, device=DEV)
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    spc.spc_conv_forward(km, Fg[:, 32:], Wg, 32, 48, out=big[:, 16:64])
    ref = oracle.conv(c, c, 3, 1, F[:, 32:], W)
    got = big.cpu().numpy()
    assert _rel_err(got[:, 16:64].astype(np.float64), ref) <= 2e-3
    assert not got[:, :16].any() and not got[:, 64:].any()


def test_conv_split_fixup_and_workspace_invariant():
    """Small levels split each output tile's offsets over CTAs (in-kernel split-K fixup):
    every one of repeated calls on one ws matches Eq. (2) (fp32 atomics make the summation
    order, hence the last bit, run-dependent), and every call (OS split, WS, hybrid;
    different c_out) leaves the workspace all-zero (spc.h contract)."""
    coords = synth.make_scan(1, 0)[:3000]
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    probe = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), -1, 0)
    ws = torch.zeros(spc.spc_conv_workspace_size(probe, 256), dtype=torch.uint8, device=DEV)
    for t, flags, ci, co in ((-1, 0, 32, 64), (-1, 0, 64, 256), (0, 1, 32, 32), (2, 1, 64, 96), (-1, 1, 16, 128),
                             (-1, 8, 32, 64), (2, 9, 64, 96)):
        km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), t, flags)
        F = synth.make_features(len(c), ci, seed=ci)
        W = synth.make_weights(27, ci, co, seed=co, nnz_per_out=10)
        R = synth.make_features(len(c), co, seed=co + 1)
        Fg = torch.from_numpy(F).to(DEV).bfloat16()
        Rg = torch.from_numpy(R).to(DEV).bfloat16()
        Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
        outs = [spc.spc_conv_forward(km, Fg, Wg, ci, co, out_dtype=torch.bfloat16, residual=Rg, ws=ws)
                for _ in range(3)]
        torch.cuda.synchronize()
        assert not ws.any(), (t, ci, co)
        ref = oracle.conv(c, c, 3, 1, F, W) + R.astype(np.float64)
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        for o in outs:
            got = o.float().cpu().numpy().astype(np.float64)
            assert (np.abs(got - ref) <= ulp + 1e-5 * np.abs(ref).max()).all(), (t, ci, co)


@pytest.mark.slow
def test_full_size_c2_sampled_parity():
    """Config C2 (~100k voxels) in the launch configuration bench.py uses: full kernel
    map bit-exact, features on 2048 sampled output rows."""
    coords = synth.make_scan(2, 0)
    spec = _spec_for(coords)
    keys, perm, st = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), 2, 1)
    np.testing.assert_array_equal(spc.spc_kmap_export(km), oracle.kmap(c, c, 3, 1))
    F = synth.make_features(len(c), 64, seed=7)
    W = synth.make_weights(27, 64, 64, seed=8, nnz_per_out=10)
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(),
                               spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16()), 64, 64,
                               out_dtype=torch.float32)
    rows = np.random.default_rng(0).choice(len(c), 2048, replace=False)
    ref = oracle.conv_rows(c, c, rows, 3, 1, F, W)
    assert _rel_err(out.cpu().numpy()[rows].astype(np.float64), ref) <= 2e-3


@pytest.mark.parametrize("c_in,c_out,dt,res,n_cut", [(16, 32, "bf16", False, 5000), (48, 96, "bf16", True, 4097),
                                                      (128, 64, "f16", True, 6000), (96, 384, "bf16", False, 3001),
                                                      (384, 256, "bf16", True, 2500)])
def test_dense_tma_k1(c_in, c_out, dt, res, n_cut):
    """A11: a K = 1 submanifold layer runs as one dense TMA-fed tcgen05 GEMM (no gather):
    BK 16/32/64 (32B/64B/128B swizzle), C_out tiled (384 = 2 x 192), ragged row tails,
    fused residual, bf16/f16 output within one ulp of the fp64 reference."""
    coords = synth.make_scan(1, 0)[:n_cut]
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(1, 1, 1, 1, 0), -1, 0)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float16
    F = synth.make_features(len(c), c_in, seed=c_in, dtype=dt)
    W = synth.make_weights(1, c_in, c_out, seed=c_out, nnz_per_out=1, dtype=dt)
    R = synth.make_features(len(c), c_out, seed=3, dtype=dt) if res else None
    big = torch.zeros(len(c), c_in + 16, dtype=tdt, device=DEV)      # read a column slice (ld_in > c_in)
    big[:, 16:] = torch.from_numpy(F).to(DEV).to(tdt)
    out = spc.spc_conv_forward(km, big[:, 16:], spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).to(tdt)), c_in,
                               c_out, out_dtype=tdt,
                               residual=None if R is None else torch.from_numpy(R).to(DEV).to(tdt))
    torch.cuda.synchronize()
    ref = F.astype(np.float64) @ W[0].astype(np.float64)
    if R is not None:
        ref = ref + R.astype(np.float64)
    got = out.float().cpu().numpy().astype(np.float64)
    mant = 7 if dt == "bf16" else 10
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - mant)
    assert (np.abs(got - ref) <= ulp + 1e-5 * np.abs(ref).max()).all()


@pytest.mark.parametrize("c_in,c_out,K,halve", [(32, 32, 3, 1), (256, 256, 3, 1), (64, 96, 5, 1), (32, 64, 3, 0)])
def test_dense_centre_initialises_ws_accumulator(c_in, c_out, K, halve):
    """SPC_OPT_CONV_DENSE_CENTRE: the centre of an all-WS submanifold map as the dense
    TMA GEMM that initialises the fp32 accumulator; the WS lists add the rest."""
    coords = synth.make_scan(1, 0)[:5000]
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(K, 1, 1, 1, 0), 0, halve)
    F = synth.make_features(len(c), c_in, seed=c_in)
    W = synth.make_weights(K ** 3, c_in, c_out, seed=c_out, nnz_per_out=10)
    R = synth.make_features(len(c), c_out, seed=4)
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    try:
        spc.spc_set_option(spc.SPC_OPT_CONV_DENSE_CENTRE, 1)
        o32 = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(), Wg, c_in, c_out, out_dtype=torch.float32)
        o16 = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(), Wg, c_in, c_out,
                                   out_dtype=torch.bfloat16, residual=torch.from_numpy(R).to(DEV).bfloat16())
        torch.cuda.synchronize()
    finally:
        spc.spc_set_option(spc.SPC_OPT_CONV_DENSE_CENTRE, -1)
    ref = oracle.conv(c, c, K, 1, F, W)
    assert _rel_err(o32.cpu().numpy().astype(np.float64), ref) <= 2e-3
    ref16 = ref + R.astype(np.float64)
    got = o16.float().cpu().numpy().astype(np.float64)
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref16), 1e-30))) - 7)
    assert (np.abs(got - ref16) <= ulp + 1e-5 * np.abs(ref16).max()).all()


@pytest.mark.parametrize("bulk", [1, 0])
@pytest.mark.parametrize("c_in,c_out,t", [(64, 64, 0), (128, 256, 0), (32, 96, 2)])
def test_ws_epilogue_variants_and_workspace_contract(bulk, c_in, c_out, t):
    """The weight-stationary scatter (bulk reductions or red.global.add) gives the
    oracle's result with a residual and leaves the caller's workspace all-zero (spc.h), so
    the next call on the same workspace is right too."""
    coords = synth.make_scan(1, 0)[:7000]
    spec = _spec_for(coords)
    keys, _, _ = _pack_sort(coords, spec)
    c = oracle.sort_coords(coords)[0]
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), t, 1)
    F = synth.make_features(len(c), c_in, seed=c_in + 1)
    W = synth.make_weights(27, c_in, c_out, seed=c_out + 2, nnz_per_out=8)
    R = synth.make_features(len(c), c_out, seed=5)
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    ws = torch.zeros(spc.spc_conv_workspace_size(km, c_out, torch.bfloat16), dtype=torch.uint8, device=DEV)
    ref = oracle.conv(c, c, 3, 1, F, W) + R.astype(np.float64)
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
    try:
        spc.spc_set_option(spc.SPC_OPT_CONV_BULK_RED, bulk)
        for _ in range(2):
            o = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(), Wg, c_in, c_out,
                                     out_dtype=torch.bfloat16, residual=torch.from_numpy(R).to(DEV).bfloat16(), ws=ws)
            torch.cuda.synchronize()
            got = o.float().cpu().numpy().astype(np.float64)
            assert (np.abs(got - ref) <= ulp + 1e-5 * np.abs(ref).max()).all()
            assert int(torch.count_nonzero(ws)) == 0
    finally:
        spc.spc_set_option(spc.SPC_OPT_CONV_BULK_RED, -1)
