"""Pins for the CPU oracle (oracle/): each test checks the oracle against something
other than itself -- brute force, Python/torch library routines, closed forms stated
in PAPER.md, the paper's worked example, and invariants.  CPU only (-m "not gpu")."""
import itertools
import os

import numpy as np
import pytest
import torch

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------------------
# canonical order
# ---------------------------------------------------------------------------------------

def test_sort_matches_python_sorted():
    rng = np.random.default_rng(1)
    c = rng.integers(-5, 5, (3000, 4)).astype(np.int32)     # many duplicates on purpose
    s, perm, dups = oracle.sort_coords(c)
    ref = sorted(range(len(c)), key=lambda i: (tuple(c[i]), i))
    assert perm.tolist() == ref
    assert np.array_equal(s, c[ref])
    assert dups == len(c) - len({tuple(r) for r in c.tolist()})


# ---------------------------------------------------------------------------------------
# packed key A1 (§5.3, readings A3/A5/A6)
# ---------------------------------------------------------------------------------------

BITS = (3, 12, 12, 8)


def _bias(b):
    return 1 << (b - 1)


def test_pack_field_positions():
    # SPEC S:96-97 style examples, shifted by the per-field bias 2^(b-1) (reading A3)
    Bb, Bx, By, Bz = BITS
    base = np.array([[0, 0, 0, 0]], np.int32)
    k0 = int(oracle.pack(base, BITS)[0][0])
    assert k0 == (_bias(Bx) << (By + Bz)) | (_bias(By) << Bz) | _bias(Bz)
    for d, step in ((0, 1 << (Bx + By + Bz)), (1, 1 << (By + Bz)), (2, 1 << Bz), (3, 1)):
        v = base.copy()
        v[0, d] = 1
        assert int(oracle.pack(v, BITS)[0][0]) - k0 == step
    lo = np.array([[0, -_bias(Bx), -_bias(By), -_bias(Bz)]], np.int32)
    assert int(oracle.pack(lo, BITS)[0][0]) == 0


def test_pack_order_preservation():
    # p_i > p_j  <=>  packed(p_i) > packed(p_j)
    c = synth.random_cloud(5000, 200, seed=3, n_batch=4)
    keys, bad = oracle.pack(c, BITS)
    assert bad == 0
    by_key = np.argsort(keys, kind="stable")
    by_tuple = sorted(range(len(c)), key=lambda i: tuple(c[i]))
    assert by_key.tolist() == by_tuple


def test_pack_out_of_range_detected():
    c = np.array([[0, 2048, 0, 0], [0, 0, -2049, 0], [0, 0, 0, 128], [8, 0, 0, 0], [0, 2047, -2048, 127]],
                 np.int32)
    keys, bad = oracle.pack(c, BITS)
    assert bad == 4 and int(keys[4]) != 0


@pytest.mark.parametrize("K", [3, 5])
def test_packed_addition_identity_exhaustive(K):
    # packed(q) + packed(delta) = packed(q + delta), exhaustive on a 16^3 grid
    Bb, Bx, By, Bz = BITS
    g = np.array(list(itertools.product(range(-8, 8), repeat=3)), np.int32)
    q = np.concatenate([np.zeros((len(g), 1), np.int32), g], 1)
    kq, _ = oracle.pack(q, BITS)
    r = (K - 1) // 2
    for dx, dy, dz in itertools.product(range(-r, r + 1), repeat=3):
        pd = dx * (1 << (By + Bz)) + dy * (1 << Bz) + dz          # the linear map
        kd, bad = oracle.pack(q + np.array([0, dx, dy, dz], np.int32), BITS)
        assert bad == 0
        assert np.array_equal((kq.astype(np.int64) + pd).astype(np.uint64), kd)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_mask_identity_matches_floor(m):
    # AND with the mask (b_i - m ones, then m zeros, per field) realises Eq. (1)
    # for s_q = 2^m; with the 2^(b-1) bias this equals floor toward -inf (reading A3).
    Bb, Bx, By, Bz = BITS
    c = synth.random_cloud(4000, 250, seed=10 + m, n_batch=8)
    keys, bad = oracle.pack(c, BITS)
    assert bad == 0
    mask = ((1 << Bb) - 1) << (Bx + By + Bz)
    for bits, sh in ((Bx, By + Bz), (By, Bz), (Bz, 0)):
        if bits > m:
            mask |= (((1 << (bits - m)) - 1) << m) << sh
    s = 1 << m
    rounded = c.copy()
    rounded[:, 1:] = np.floor_divide(c[:, 1:], s) * s
    kr, bad = oracle.pack(rounded, BITS)
    assert bad == 0
    assert np.array_equal(keys & np.uint64(mask), kr)


# ---------------------------------------------------------------------------------------
# Eq. (1) / Eq. (3)
# ---------------------------------------------------------------------------------------

def test_round_down_is_floor():
    for v in range(-40, 41):
        for s in (1, 2, 4, 8, 16):
            assert oracle.round_down(v, s) == (v // s) * s        # Python // floors


def test_downsample_examples():
    # {(2,2,2),(3,3,3)} with s=4 -> {(0,0,0)};  S:459: (5,3,7), s=4 -> (4,0,4)
    out = oracle.downsample(np.array([[0, 2, 2, 2], [0, 3, 3, 3]]), 4)
    assert out.tolist() == [[0, 0, 0, 0]]
    assert oracle.downsample(np.array([[0, 5, 3, 7]]), 4).tolist() == [[0, 4, 0, 4]]
    assert oracle.downsample(np.array([[1, -1, -3, -4]]), 2).tolist() == [[1, -2, -4, -4]]


def test_downsample_matches_set_comprehension():
    c = synth.random_cloud(3000, 300, seed=5, n_batch=3)
    for s in (2, 4, 8, 16):
        ref = sorted({(b, (x // s) * s, (y // s) * s, (z // s) * s) for b, x, y, z in c.tolist()})
        assert oracle.downsample(c, s).tolist() == [list(t) for t in ref]


def test_eq3_closed_form_equals_recursive():
    # V_i = floor(V_{i-1}/2^i) 2^i ... = floor(V_0/2^i) 2^i
    c = synth.surface_cloud(5000, seed=7, n_batch=2, scale=3.0)
    v = oracle.sort_coords(c)[0]
    for i in range(1, 6):
        v = oracle.downsample(v, 2 ** i)
        assert np.array_equal(v, oracle.downsample(c, 2 ** i))


# ---------------------------------------------------------------------------------------
# offsets and the hybrid partition
# ---------------------------------------------------------------------------------------

def test_offsets_delta_5_2():
    off, l1 = oracle.offsets(5, 2)
    assert set(map(tuple, off.tolist())) == set(itertools.product((-4, -2, 0, 2, 4), repeat=3))
    assert off.tolist() == sorted(off.tolist())                    # lexicographic, dz fastest


def test_offsets_group0_and_mirror():
    off, l1 = oracle.offsets(3, 1)
    assert off[:3].tolist() == [[-1, -1, -1], [-1, -1, 0], [-1, -1, 1]]   # P:266 group 0
    for K in (1, 3, 5):
        off, l1 = oracle.offsets(K, 1)
        kv = K ** 3
        for k in range(kv):
            assert (off[kv - 1 - k] == -off[k]).all()                      # mirror(k) = K^3-1-k
        assert (off[(kv - 1) // 2] == 0).all()
        assert l1.max() == 3 * (K - 1) // 2                                # P:207 L1NormMax/s_p


def test_hybrid_partition_counts():
    _, l1 = oracle.offsets(5, 1)
    assert int((l1 < 3).sum()) == 25 and int((l1 >= 3).sum()) == 100
    assert int((l1 < 5).sum()) == 93                                      # P:570 ("at least 93")
    for K, n_hybrid in ((3, 3), (5, 6)):
        _, l1 = oracle.offsets(K, 1)
        ts = [t for t in range(0, l1.max() + 2) if 0 < t <= l1.max()]
        assert len(ts) == n_hybrid
        assert int((l1 < l1.max() + 1).sum()) == K ** 3 and int((l1 < 0).sum()) == 0


def test_even_kernel_rejected():
    with pytest.raises(ValueError):
        oracle.offsets(2, 1)


# ---------------------------------------------------------------------------------------
# kernel map -- brute force, paper example, invariants
# ---------------------------------------------------------------------------------------

def _brute_kmap(inp, out, K, spacing, transposed=False):
    r = (K - 1) // 2
    offs = [np.array(o) * spacing for o in itertools.product(range(-r, r + 1), repeat=3)]
    res = []
    for k, o in enumerate(offs):
        for i in range(len(out)):
            for j in range(len(inp)):
                q = out[i, 1:] - o if transposed else out[i, 1:] + o
                if inp[j, 0] == out[i, 0] and (inp[j, 1:] == q).all():
                    res.append((k, i, j))
    return sorted(res)


def test_paper_worked_example():
    lines = [l.split() for l in open(os.path.join(HERE, "golden", "zdelta_worked_example.txt"))
             if l.strip() and not l.startswith("#")]
    K = int(next(l[1] for l in lines if l[0] == "K"))
    sp = int(next(l[1] for l in lines if l[0] == "spacing"))
    out = np.array([[0] + [int(v) for v in l[1:]] for l in lines if l[0] == "output"], np.int32)
    inp = np.array([[0] + [int(v) for v in l[1:]] for l in lines if l[0] == "input"], np.int32)
    exp = [[int(v) for v in l[1:]] for l in lines if l[0] == "triple"]
    assert oracle.kmap(inp, out, K, sp).tolist() == exp


@pytest.mark.parametrize("K,sp,kind", [(1, 1, "subm"), (3, 1, "subm"), (5, 1, "subm"), (3, 2, "subm"),
                                       (3, 1, "strided"), (5, 1, "strided"), (3, 2, "strided"),
                                       (3, 1, "transposed"), (5, 2, "transposed")])
def test_kmap_matches_brute_force(K, sp, kind):
    c = synth.random_cloud(140, 9, seed=K * 10 + sp, n_batch=2) * np.array([1, sp, sp, sp], np.int32)
    fine = oracle.sort_coords(c)[0]
    if kind == "subm":
        inp = out = fine
        got = oracle.kmap(inp, out, K, sp)
        ref = _brute_kmap(inp, out, K, sp)
    else:
        coarse = oracle.downsample(fine, 2 * sp)
        if kind == "strided":
            got = oracle.kmap(fine, coarse, K, sp)
            ref = _brute_kmap(fine, coarse, K, sp)
        else:
            got = oracle.kmap(coarse, fine, K, sp, transposed=True)
            ref = _brute_kmap(coarse, fine, K, sp, transposed=True)
    assert [tuple(t) for t in got.tolist()] == ref
    assert len(ref) > 0


def test_kmap_invariants():
    c = oracle.sort_coords(synth.surface_cloud(3000, seed=11, n_batch=2))[0]
    for K in (3, 5):
        kv = K ** 3
        t = oracle.kmap(c, c, K, 1)
        centre = t[t[:, 0] == (kv - 1) // 2]
        assert (centre[:, 1] == centre[:, 2]).all() and len(centre) == len(c)
        a = {tuple(x) for x in t.tolist()}
        b = {(kv - 1 - k, j, i) for k, i, j in t.tolist()}
        assert a == b
        # batch isolation
        assert (c[t[:, 1], 0] == c[t[:, 2], 0]).all()
    coarse = oracle.downsample(c, 2)
    s = oracle.kmap(c, coarse, 3, 1)
    tr = oracle.kmap(coarse, c, 3, 1, transposed=True)
    assert sorted(map(tuple, s[:, [0, 2, 1]].tolist())) == list(map(tuple, tr.tolist()))
    assert set(s[:, 2].tolist()) == set(range(len(c)))        # every fine voxel has a parent
    assert set(s[:, 1].tolist()) == set(range(len(coarse)))   # no empty output rows
    # translation by a multiple of the largest stride leaves the map unchanged
    sh = c + np.array([0, 32, -64, 16], np.int32)
    assert np.array_equal(oracle.kmap(sh, sh, 3, 1), oracle.kmap(c, c, 3, 1))


# ---------------------------------------------------------------------------------------
# Eq. (2) in fp64 -- torch conv3d (library routine) on the dense grid, special cases
# ---------------------------------------------------------------------------------------

def _dense_weight(W, K):
    # weight[co, ci, ex+r, ey+r, ez+r] = W[k(e), ci, co]
    kv, ci, co = W.shape
    return torch.from_numpy(W.reshape(K, K, K, ci, co)).permute(4, 3, 0, 1, 2).contiguous()


def _grid(coords, C, F, origin, size):
    g = torch.zeros((1, C) + size, dtype=torch.float64)
    for r, (b, x, y, z) in enumerate(coords.tolist()):
        g[0, :, x - origin[0], y - origin[1], z - origin[2]] = torch.from_numpy(F[r])
    return g


@pytest.mark.parametrize("K,sp", [(1, 1), (3, 1), (5, 1), (3, 2)])
def test_conv_submanifold_vs_conv3d(K, sp):
    rng = np.random.default_rng(K + 7 * sp)
    c = oracle.sort_coords(synth.random_cloud(120, 7, seed=K + 3 * sp, signed=False)
                           * np.array([1, sp, sp, sp], np.int32))[0]
    F = rng.uniform(-1, 1, (len(c), 5))
    W = rng.uniform(-1, 1, (K ** 3, 5, 6))
    got = oracle.conv(c, c, K, sp, F, W)
    # compress the s_p lattice: a stride-s_p layer on V is a stride-1 layer on V/s_p
    cc = c.copy()
    cc[:, 1:] //= sp
    r = (K - 1) // 2
    g = _grid(cc, 5, F, (0, 0, 0), (8, 8, 8))
    y = torch.nn.functional.conv3d(g, _dense_weight(W, K), padding=r)
    ref = np.stack([y[0, :, x, yy, z].numpy() for _, x, yy, z in cc.tolist()])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K", [3, 5])
def test_conv_strided_and_transposed_vs_torch(K):
    rng = np.random.default_rng(K)
    c = oracle.sort_coords(synth.random_cloud(150, 8, seed=K, signed=False))[0]
    coarse = oracle.downsample(c, 2)
    r = (K - 1) // 2
    F = rng.uniform(-1, 1, (len(c), 4))
    W = rng.uniform(-1, 1, (K ** 3, 4, 3))
    got = oracle.conv(c, coarse, K, 1, F, W)
    g = _grid(c, 4, F, (0, 0, 0), (8, 8, 8))
    y = torch.nn.functional.conv3d(g, _dense_weight(W, K), stride=2, padding=r)
    ref = np.stack([y[0, :, x // 2, yy // 2, z // 2].numpy() for _, x, yy, z in coarse.tolist()])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    # transposed: coarse in -> fine out, same weight index as the strided layer
    Fc = rng.uniform(-1, 1, (len(coarse), 4))
    got_t = oracle.conv(coarse, c, K, 1, Fc, W, transposed=True)
    gc = torch.zeros((1, 4, 4, 4, 4), dtype=torch.float64)
    for rr, (_, x, yy, z) in enumerate(coarse.tolist()):
        gc[0, :, x // 2, yy // 2, z // 2] = torch.from_numpy(Fc[rr])
    wt = torch.from_numpy(W.reshape(K, K, K, 4, 3)).permute(3, 4, 0, 1, 2).contiguous()
    yt = torch.nn.functional.conv_transpose3d(gc, wt, stride=2, padding=r, output_padding=1)
    ref_t = np.stack([yt[0, :, x, yy, z].numpy() for _, x, yy, z in c.tolist()])
    np.testing.assert_allclose(got_t, ref_t, rtol=1e-12, atol=1e-12)


def test_conv_special_cases():
    rng = np.random.default_rng(0)
    c = oracle.sort_coords(synth.surface_cloud(800, seed=2))[0]
    F = rng.uniform(-1, 1, (len(c), 8))
    # K=1, W=I -> identity
    np.testing.assert_array_equal(oracle.conv(c, c, 1, 1, F, np.eye(8)[None]), F)
    # single voxel -> F W_centre
    W = rng.uniform(-1, 1, (27, 8, 4))
    one = c[:1]
    np.testing.assert_allclose(oracle.conv(one, one, 3, 1, F[:1], W), F[:1] @ W[13], rtol=1e-14)
    # W = 0 -> 0; linearity; OS order == WS order (north_star invariant)
    assert not oracle.conv(c, c, 3, 1, F, np.zeros_like(W)).any()
    a = oracle.conv(c, c, 3, 1, F, W, order="os")
    b = oracle.conv(c, c, 3, 1, F, W, order="ws")
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv(c, c, 3, 1, 2.5 * F, W), 2.5 * a, rtol=1e-12, atol=1e-12)
    rows = np.array([0, 5, len(c) - 1])
    np.testing.assert_allclose(oracle.conv_rows(c, c, rows, 3, 1, F, W), a[rows], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("K", [3, 5])
def test_conv_dilated_off_lattice_vs_conv3d(K):
    """Dilation d = 2 on coordinates that are NOT on a 2-lattice (VERDICT r1 pin gap):
    submanifold = conv3d(dilation=2, padding=2r); strided = conv3d(stride=2, dilation=2)
    at the Eq. (1) sites; transposed = conv_transpose3d(stride=2, dilation=2)."""
    d = 2
    rng = np.random.default_rng(40 + K)
    c = oracle.sort_coords(synth.random_cloud(160, 8, seed=50 + K, signed=False))[0]
    r = (K - 1) // 2
    F = rng.uniform(-1, 1, (len(c), 4))
    W = rng.uniform(-1, 1, (K ** 3, 4, 3))
    g = _grid(c, 4, F, (0, 0, 0), (8, 8, 8))
    # submanifold, spacing = tensor stride 1 x dilation 2
    got = oracle.conv(c, c, K, d, F, W)
    y = torch.nn.functional.conv3d(g, _dense_weight(W, K), padding=r * d, dilation=d)
    ref = np.stack([y[0, :, x, yy, z].numpy() for _, x, yy, z in c.tolist()])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    # strided
    coarse = oracle.downsample(c, 2)
    got_s = oracle.conv(c, coarse, K, d, F, W)
    ys = torch.nn.functional.conv3d(g, _dense_weight(W, K), stride=2, padding=r * d, dilation=d)
    ref_s = np.stack([ys[0, :, x // 2, yy // 2, z // 2].numpy() for _, x, yy, z in coarse.tolist()])
    np.testing.assert_allclose(got_s, ref_s, rtol=1e-12, atol=1e-12)
    # transposed (same weight index as the strided layer)
    Fc = rng.uniform(-1, 1, (len(coarse), 4))
    got_t = oracle.conv(coarse, c, K, d, Fc, W, transposed=True)
    gc = torch.zeros((1, 4, 4, 4, 4), dtype=torch.float64)
    for rr, (_, x, yy, z) in enumerate(coarse.tolist()):
        gc[0, :, x // 2, yy // 2, z // 2] = torch.from_numpy(Fc[rr])
    wt = torch.from_numpy(W.reshape(K, K, K, 4, 3)).permute(3, 4, 0, 1, 2).contiguous()
    yt = torch.nn.functional.conv_transpose3d(gc, wt, stride=2, padding=r * d, dilation=d,
                                              output_padding=8 - (3 * 2 - 2 * r * d + d * (K - 1) + 1))
    ref_t = np.stack([yt[0, :, x, yy, z].numpy() for _, x, yy, z in c.tolist()])
    np.testing.assert_allclose(got_t, ref_t, rtol=1e-12, atol=1e-12)


def test_openmp_build_is_bit_identical():
    """The OpenMP oracle build (cpu_baseline timing) computes every Eq. (2) row in the same
    order as the plain build: results are bit-identical."""
    rng = np.random.default_rng(5)
    c = oracle.sort_coords(synth.surface_cloud(3000, seed=4))[0]
    F = rng.uniform(-1, 1, (len(c), 16))
    W = rng.uniform(-1, 1, (27, 16, 8))
    rows = rng.choice(len(c), 500, replace=False)
    a, ar = oracle.conv(c, c, 3, 1, F, W), oracle.conv_rows(c, c, rows, 3, 1, F, W)
    try:
        oracle.use_openmp(True)
        b, br = oracle.conv(c, c, 3, 1, F, W), oracle.conv_rows(c, c, rows, 3, 1, F, W)
    finally:
        oracle.use_openmp(False)
    assert np.array_equal(a, b) and np.array_equal(ar, br)


# ---------------------------------------------------------------------------------------
# voxelization: P:96 v = floor(p / g); S:70-78 quantize; S:132 averaging
# ---------------------------------------------------------------------------------------

def test_voxelize_spec_examples():
    """(1.25, -0.30, 0.999) at g = 0.5 -> (2, -1, 1) (floor(-0.6) = -1, not
    truncation); the origin maps to the origin for any g."""
    c, pv, _ = oracle.voxelize(np.array([[1.25, -0.30, 0.999]], np.float32), (0.5, 0.5, 0.5))
    assert c.tolist() == [[0, 2, -1, 1]] and pv.tolist() == [0]
    c, _, _ = oracle.voxelize(np.zeros((1, 3), np.float32), (0.05, 0.1, 0.2))
    assert c.tolist() == [[0, 0, 0, 0]]


def test_voxelize_matches_set_bruteforce():
    """random points in a 10 m cube at g = 0.1: the voxel set is the set of floored
    triples (Python set over math.floor of numpy float32 quotients), canonical order is
    Python's tuple sort, every point's index points at its own voxel, and each mean is
    the plain Python mean of the voxel's features in point order (bit-equal)."""
    import math
    rng = np.random.default_rng(11)
    n = 1000
    P = rng.uniform(-5, 5, (n, 3)).astype(np.float32)
    P[::7] = P[3]                       # repeated points (merged voxels)
    b = rng.integers(0, 3, n).astype(np.int32)
    F = rng.uniform(-1, 1, (n, 5)).astype(np.float32)
    g = np.float32(0.1)
    vox = [(int(b[i]),) + tuple(math.floor(float(P[i, d] / g)) for d in range(3)) for i in range(n)]
    ref = sorted(set(vox))
    c, pv, m = oracle.voxelize(P, (0.1, 0.1, 0.1), batch=b, feats=F)
    assert [tuple(r) for r in c.tolist()] == ref
    assert all(tuple(c[pv[i]].tolist()) == vox[i] for i in range(n))
    members = {}
    for i in range(n):
        members.setdefault(vox[i], []).append(i)
    for v, rows in members.items():
        for ch in range(5):
            s = 0.0
            for i in rows:
                s += float(F[i, ch])
            assert m[ref.index(v), ch] == s / len(rows)


def test_voxelize_boundaries_and_negatives():
    """Points exactly on grid planes belong to the voxel above (floor of an exact
    quotient); tiny negative values floor to -1; a repeated point's mean is itself."""
    P = np.array([[-0.5, 0.25, 0.0], [-1e-8, 1e-8, -0.25], [0.75, -0.75, 2.5], [0.75, -0.75, 2.5]], np.float32)
    F = np.array([[1.0], [2.0], [3.0], [5.0]], np.float32)
    c, pv, m = oracle.voxelize(P, (0.25, 0.25, 0.25), feats=F)
    assert c.tolist() == [[0, -2, 1, 0], [0, -1, 0, -1], [0, 3, -3, 10]]
    assert pv.tolist() == [0, 1, 2, 2]
    assert m[:, 0].tolist() == [1.0, 2.0, 4.0]


def test_voxelize_rejects_non_finite():
    """a non-finite point is rejected with a diagnostic naming its index."""
    P = np.zeros((10, 3), np.float32)
    P[7, 1] = np.nan
    with pytest.raises(ValueError, match="point 7"):
        oracle.voxelize(P, (0.1, 0.1, 0.1))
    P[7, 1] = 0
    P[3, 2] = np.inf
    with pytest.raises(ValueError, match="point 3"):
        oracle.voxelize(P, (0.1, 0.1, 0.1))


# ---------------------------------------------------------------------------------------
# (Kx, Ky, Kz) offset boxes, even sizes {0..K-1} (reading E1), and spconv's
# regular output rule
# ---------------------------------------------------------------------------------------

def _box_offsets_py(K, spacing):
    rng = [range(-(k - 1) // 2, (k - 1) // 2 + 1) if k % 2 else range(0, k) for k in K]
    return [(ex * spacing, ey * spacing, ez * spacing) for ex in rng[0] for ey in rng[1] for ez in rng[2]]


@pytest.mark.parametrize("K,stride,transposed", [((2, 2, 2), 2, False), ((2, 2, 2), 2, True), ((3, 1, 1), 1, False),
                                                 ((1, 3, 1), 1, False), ((3, 3, 1), 2, False), ((4, 2, 3), 1, False)])
def test_box_kmap_bruteforce(K, stride, transposed):
    """orc_kmap3 vs an O(N^2 kv) double loop over explicitly enumerated offsets."""
    fine = oracle.sort_coords(synth.random_cloud(300, 10, seed=sum(K) + stride, n_batch=2))[0]
    coarse = oracle.downsample(fine, stride) if stride > 1 else fine
    inp, out = (coarse, fine) if transposed else (fine, coarse)
    off = _box_offsets_py(K, 1)
    ref = []
    for k, d in enumerate(off):
        for i, q in enumerate(out.tolist()):
            t = [q[0]] + [q[1 + a] - d[a] if transposed else q[1 + a] + d[a] for a in range(3)]
            for j, p in enumerate(inp.tolist()):
                if p == t:
                    ref.append((k, i, j))
    got = oracle.kmap(inp, out, K, 1, transposed=transposed)
    assert [tuple(r) for r in got.tolist()] == sorted(ref)


def test_box_conv_matches_torch_conv3d():
    """K = 2 stride-2 down (conv3d kernel 2 stride 2), its transposed up
    (conv_transpose3d), and a non-cubic (3, 1, 1) submanifold layer (conv3d padding
    (1, 0, 0)) on dense grids in float64, read at the sparse sites."""
    rng = np.random.default_rng(21)
    n = 8
    occ = rng.random((n, n, n)) < 0.4
    fine = np.array([[0, x, y, z] for x, y, z in zip(*np.nonzero(occ))], np.int32)
    F = rng.uniform(-1, 1, (len(fine), 3))
    grid = torch.zeros((1, 3, n, n, n), dtype=torch.float64)
    for r, (_, x, y, z) in enumerate(fine.tolist()):
        grid[0, :, x, y, z] = torch.from_numpy(F[r])
    # down: out sites = Eq. (1) stride-2 sites (= the regular rule for K = 2, s = 2)
    coarse = oracle.downsample(fine, 2)
    W = rng.uniform(-1, 1, (8, 3, 4))
    got = oracle.conv(fine, coarse, (2, 2, 2), 1, F, W)
    w = torch.from_numpy(W.reshape(2, 2, 2, 3, 4)).permute(4, 3, 0, 1, 2).contiguous()
    y = torch.nn.functional.conv3d(grid, w, stride=2)
    ref = np.stack([y[0, :, x // 2, yy // 2, z // 2].numpy() for _, x, yy, z in coarse.tolist()])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    # up (transposed, same weight index): fine outputs from coarse inputs
    Fc = rng.uniform(-1, 1, (len(coarse), 4))
    Wt = rng.uniform(-1, 1, (8, 4, 3))
    got_t = oracle.conv(coarse, fine, (2, 2, 2), 1, Fc, Wt, transposed=True)
    gc = torch.zeros((1, 4, n // 2, n // 2, n // 2), dtype=torch.float64)
    for r, (_, x, yy, z) in enumerate(coarse.tolist()):
        gc[0, :, x // 2, yy // 2, z // 2] = torch.from_numpy(Fc[r])
    wt = torch.from_numpy(Wt.reshape(2, 2, 2, 4, 3)).permute(3, 4, 0, 1, 2).contiguous()
    yt = torch.nn.functional.conv_transpose3d(gc, wt, stride=2)
    ref_t = np.stack([yt[0, :, x, yy, z].numpy() for _, x, yy, z in fine.tolist()])
    np.testing.assert_allclose(got_t, ref_t, rtol=1e-12, atol=1e-12)
    # non-cubic submanifold (3, 1, 1)
    W3 = rng.uniform(-1, 1, (3, 3, 2))
    got3 = oracle.conv(fine, fine, (3, 1, 1), 1, F, W3)
    w3 = torch.from_numpy(W3.reshape(3, 1, 1, 3, 2)).permute(4, 3, 0, 1, 2).contiguous()
    y3 = torch.nn.functional.conv3d(grid, w3, padding=(1, 0, 0))
    ref3 = np.stack([y3[0, :, x, yy, z].numpy() for _, x, yy, z in fine.tolist()])
    np.testing.assert_allclose(got3, ref3, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,s", [(3, 2), (3, 1), ((3, 1, 1), 2), (5, 2)])
def test_regular_outputs_is_conv_support(K, s):
    """spconv's regular rule = the support of conv3d(occupancy, ones, stride s, padding
    (K-1)/2): a site is an output iff its kernel footprint touches an input."""
    rng = np.random.default_rng(4)
    n = 12
    occ = np.zeros((n, n, n), bool)
    occ[2:10, 2:10, 2:10] = rng.random((8, 8, 8)) < 0.05
    fine = np.array([[0, x, y, z] for x, y, z in zip(*np.nonzero(occ))], np.int32)
    kx, ky, kz = K if isinstance(K, tuple) else (K, K, K)
    got = oracle.regular_outputs(fine, K, 1, s)
    ones = torch.ones((1, 1, kx, ky, kz), dtype=torch.float64)
    sup = torch.nn.functional.conv3d(torch.from_numpy(occ.astype(np.float64))[None, None], ones, stride=s,
                                     padding=((kx - 1) // 2, (ky - 1) // 2, (kz - 1) // 2))[0, 0].numpy() > 0
    ref = sorted((0, int(x) * s, int(y) * s, int(z) * s) for x, y, z in zip(*np.nonzero(sup)))
    assert [tuple(r) for r in got.tolist()] == ref


def test_regular_outputs_k2_s2_equals_eq1_downsample():
    """K = 2, s = 2 (offsets {0, 1}^3): every point has exactly one lattice site p - delta,
    its Eq. (1) parent, so the regular rule and Eq. (1) give the same sites."""
    c = oracle.sort_coords(synth.random_cloud(2000, 40, seed=8, n_batch=3))[0]
    assert np.array_equal(oracle.regular_outputs(c, (2, 2, 2), 1, 2), oracle.downsample(c, 2))
