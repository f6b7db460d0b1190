"""GPU parity of the SURVEY NEXT-4 additions through the C ABI against the CPU oracle:
the fused BN / residual / ReLU epilogue (spc_conv_forward_ex, spc_bn_fold), the data
gradient (forward kernels on the dgrad map with spc_prepare_weight_ex) and the weight
gradient (spc_conv_wgrad, tcgen05 with MN-major operands; FFMA for fp32).

Tolerances as north_star's for features: max|gpu - ref| <= 2e-3 * max|ref| for f16/bf16
inputs with fp32 outputs, <= 1e-5 * max|ref| for the fp32 path."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"
TDT = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}


def _spec_for(coords, max_stride=16, reach=16):
    return spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), int(coords[:, 0].max()) + 1, max_stride,
                             reach)


def _keys(c_sorted, spec):
    k, bad = oracle.pack(c_sorted, spec.astuple())
    assert bad == 0
    return torch.from_numpy(k.view(np.int64)).to(DEV)


def _case(n=6000, seed=0):
    coords = synth.make_scan(1, seed)[:n]
    spec = _spec_for(coords)
    fine = oracle.sort_coords(coords)[0]
    coarse = oracle.downsample(coords, 2)
    return spec, fine, coarse


def _rel(got, ref):
    m = np.abs(ref).max()
    return float(np.abs(got - ref).max() / (m if m > 0 else 1.0))


def _map(a, b, spec, geom, t, flags):
    ka = _keys(a, spec)
    return spc.spc_build_kmap(ka, ka if a is b else _keys(b, spec), spec, geom, t, flags)


def _layer(kind, K, spec, fine, coarse):
    """(in coords, out coords, forward geom, dgrad geom, transposed flag) of a layer kind."""
    if kind == "subm":
        return fine, fine, spc.Geom(K, 1, 1, 1, 0), None, False
    if kind == "strided":
        return fine, coarse, spc.Geom(K, 2, 1, 1, 0), spc.Geom(K, 2, 1, 1, 1), False
    return coarse, fine, spc.Geom(K, 2, 1, 1, 1), spc.Geom(K, 2, 1, 1, 0), True


# ---------------------------------------------------------------------------------------
# fused epilogue
# ---------------------------------------------------------------------------------------

EPI_CASES = [
    # (K, t, flags, c_in, c_out, dtype, out dtype, residual, relu)
    (3, -1, 0, 32, 64, "bf16", "f32", False, True),      # OS, final stores
    (3, -1, 8, 64, 64, "bf16", "bf16", True, True),      # OS density order, bf16 out + residual
    (3, 0, 1, 64, 128, "bf16", "f32", True, True),       # WS (halved) -> k_convert
    (3, 2, 1, 32, 96, "f16", "f32", False, True),        # hybrid
    (1, -1, 0, 64, 32, "bf16", "f32", True, True),       # K = 1: dense TMA GEMM epilogue
    (3, -1, 0, 256, 256, "bf16", "f32", False, False),   # BN only (no ReLU), wide OS
    (3, 2, 1, 16, 32, "f32", "f32", True, True),         # fp32 FFMA path
    (3, -1, 0, 16, 32, "f32", "f32", False, True),
]


@pytest.mark.parametrize("K,t,flags,c_in,c_out,dt,odt,res,relu", EPI_CASES)
def test_conv_epilogue_bn_residual_relu(K, t, flags, c_in, c_out, dt, odt, res, relu):
    spec, c, _ = _case(5000, seed=1)
    k = _keys(c, spec)   # halving needs one key array for in and out
    km = spc.spc_build_kmap(k, k, spec, spc.Geom(K, 1, 1, 1, 0), t, flags)
    rng = np.random.default_rng(c_in + c_out)
    F = synth.make_features(len(c), c_in, seed=3, dtype=dt)
    W = synth.make_weights(K ** 3, c_in, c_out, seed=4, nnz_per_out=8, dtype=dt)
    gamma, beta = rng.uniform(0.5, 1.5, c_out), rng.normal(0, 0.5, c_out)
    mean, var = rng.normal(0, 0.3, c_out), rng.uniform(0.5, 2.0, c_out)
    R = synth.make_features(len(c), c_out, seed=5, dtype="bf16" if odt == "bf16" else "f32") if res else None
    f32 = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(DEV)
    scale, shift = spc.spc_bn_fold(f32(gamma), f32(beta), f32(mean), f32(var), 1e-3)
    Fg = torch.from_numpy(F).to(DEV).to(TDT[dt])
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).to(TDT[dt]))
    Rg = torch.from_numpy(R).to(DEV).to(TDT[odt]) if res else None
    out = spc.spc_conv_forward(km, Fg, Wg, c_in, c_out, out_dtype=TDT[odt], residual=Rg, scale=scale, shift=shift,
                               relu=relu)
    torch.cuda.synchronize()
    ref = oracle.bn_relu(oracle.conv(c, c, K, 1, F, W), gamma, beta, mean, var, 1e-3, residual=R, relu=relu)
    got = out.float().cpu().numpy().astype(np.float64)
    if odt == "bf16":
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        assert (np.abs(got - ref) <= ulp + 2e-3 * np.abs(ref).max()).all()
    else:
        assert _rel(got, ref) <= (1e-5 if dt == "f32" else 2e-3)
    if relu:
        assert (got >= 0).all()


def test_bn_fold_matches_definition():
    rng = np.random.default_rng(0)
    g, b, m, v = rng.uniform(0.5, 2, 80), rng.normal(0, 1, 80), rng.normal(0, 1, 80), rng.uniform(0.1, 3, 80)
    f32 = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(DEV)
    s, sh = spc.spc_bn_fold(f32(g), f32(b), f32(m), f32(v), 1e-5)
    x = rng.normal(0, 2, (7, 80))
    got = x * s.cpu().numpy().astype(np.float64) + sh.cpu().numpy().astype(np.float64)
    assert _rel(got, oracle.bn_relu(x, g, b, m, v, 1e-5, relu=False)) <= 1e-6


# ---------------------------------------------------------------------------------------
# data gradient: forward kernels on the dgrad map
# ---------------------------------------------------------------------------------------

DGRAD_CASES = [
    # (K, kind, t, flags, c_in, c_out, dtype)   (c_in / c_out of the FORWARD layer)
    (3, "subm", -1, 0, 32, 64, "bf16"), (3, "subm", 0, 1, 64, 32, "bf16"), (3, "subm", 2, 1, 96, 64, "bf16"),
    (3, "subm", -1, 8, 32, 32, "bf16"), (5, "subm", 3, 1, 32, 32, "bf16"), (1, "subm", -1, 0, 64, 128, "bf16"),
    (3, "strided", -1, 0, 32, 64, "bf16"), (3, "strided", 0, 0, 64, 64, "bf16"),
    (3, "transposed", -1, 0, 64, 32, "bf16"), (3, "transposed", 2, 0, 128, 96, "bf16"),
    (3, "subm", 2, 1, 16, 32, "f32"), (3, "strided", -1, 0, 32, 16, "f32"),
]


@pytest.mark.parametrize("K,kind,t,flags,c_in,c_out,dt", DGRAD_CASES)
def test_dgrad_matches_oracle(K, kind, t, flags, c_in, c_out, dt):
    spec, fine, coarse = _case(6000, seed=2)
    a, b, g_fwd, g_bwd, tr = _layer(kind, K, spec, fine, coarse)
    G = synth.make_features(len(b), c_out, seed=7, dtype=dt)
    W = synth.make_weights(K ** 3, c_in, c_out, seed=8, nnz_per_out=8, dtype=dt)
    Wt = torch.from_numpy(W).to(DEV).to(TDT[dt])
    if kind == "subm":   # the forward map itself, W'_k = W_{K^3-1-k}^T
        km = _map(a, b, spec, g_fwd, t, flags)
        Wp = spc.spc_prepare_weight_ex(Wt, spc.SPC_WEIGHT_DGRAD_MIRROR)
    else:                # the map of the opposite direction (out = the layer's inputs), W'_k = W_k^T
        km = _map(b, a, spec, g_bwd, t, flags)
        Wp = spc.spc_prepare_weight_ex(Wt, spc.SPC_WEIGHT_DGRAD)
    dF = spc.spc_conv_forward(km, torch.from_numpy(G).to(DEV).to(TDT[dt]), Wp, c_out, c_in,
                              out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle.conv_dgrad(a, b, K, 1, G, W, transposed=tr)
    assert _rel(dF.cpu().numpy().astype(np.float64), ref) <= (1e-5 if dt == "f32" else 2e-3)


def test_prepare_weight_modes_exact():
    """The dgrad preparations are exact permutations of the forward weight: a dgrad conv
    with a one-hot weight reproduces the transposed / mirrored entry bit-exactly."""
    kv, ci, co = 27, 16, 32
    W = torch.zeros(kv, ci, co)
    W[4, 3, 17] = 1.0
    W[22, 15, 0] = -2.0
    Wt = spc.spc_prepare_weight_ex(W.to(DEV), spc.SPC_WEIGHT_DGRAD)
    Wm = spc.spc_prepare_weight_ex(W.to(DEV), spc.SPC_WEIGHT_DGRAD_MIRROR)
    torch.cuda.synchronize()
    ref_t = W.permute(0, 2, 1).contiguous()
    ref_m = ref_t.flip(0).contiguous()
    assert torch.equal(Wt.cpu().view(kv, co, ci), ref_t) and torch.equal(Wm.cpu().view(kv, co, ci), ref_m)


# ---------------------------------------------------------------------------------------
# weight gradient
# ---------------------------------------------------------------------------------------

WGRAD_CASES = [
    # (K, kind, t, flags, c_in, c_out, dtype)
    (3, "subm", -1, 0, 32, 32, "bf16"),      # all dense columns (OS table, tile-mask skipping)
    (3, "subm", -1, 8, 64, 64, "bf16"),      # density-ordered map (wgrad reads the unordered table)
    (3, "subm", 0, 1, 64, 96, "bf16"),       # halved WS lists + mirrored pairs, N padded 96 -> 128
    (3, "subm", 2, 1, 128, 128, "f16"),      # hybrid
    (3, "subm", 0, 0, 256, 256, "bf16"),     # unhalved lists, 2 c_in tiles
    (5, "subm", 3, 1, 16, 16, "bf16"),       # K = 5 hybrid, narrow (M and N zero-padded)
    (1, "subm", -1, 0, 384, 32, "bf16"),     # K = 1, 3 c_in tiles
    (3, "subm", 0, 1, 32, 384, "bf16"),      # 2 c_out tiles of 256
    (3, "strided", -1, 0, 32, 64, "bf16"), (3, "strided", 0, 0, 64, 64, "bf16"),
    (3, "transposed", -1, 0, 64, 32, "bf16"), (3, "transposed", 2, 0, 128, 96, "bf16"),
    (3, "subm", 0, 1, 16, 32, "f32"), (3, "strided", -1, 0, 32, 16, "f32"),
]


@pytest.mark.parametrize("K,kind,t,flags,c_in,c_out,dt", WGRAD_CASES)
def test_wgrad_matches_oracle(K, kind, t, flags, c_in, c_out, dt):
    spec, fine, coarse = _case(6000, seed=3)
    a, b, g_fwd, _, tr = _layer(kind, K, spec, fine, coarse)
    km = _map(a, b, spec, g_fwd, t, flags)
    F = synth.make_features(len(a), c_in, seed=11, dtype=dt)
    G = synth.make_features(len(b), c_out, seed=12, dtype=dt)
    Fg = torch.from_numpy(F).to(DEV).to(TDT[dt])
    Gg = torch.from_numpy(G).to(DEV).to(TDT[dt])
    dW = spc.spc_conv_wgrad(km, Fg, Gg, c_in, c_out)
    torch.cuda.synchronize()
    ref = oracle.conv_wgrad(a, b, K, 1, F, G, transposed=tr)
    assert _rel(dW.cpu().numpy().astype(np.float64), ref) <= (1e-5 if dt == "f32" else 2e-3)
    # accumulation contract: a second call adds the same gradient
    spc.spc_conv_wgrad(km, Fg, Gg, c_in, c_out, d_weight=dW)
    torch.cuda.synchronize()
    assert _rel(dW.cpu().numpy().astype(np.float64), 2 * ref) <= (1e-5 if dt == "f32" else 2e-3)


def test_training_step_full_c2_level0():
    """One layer's backward at C2 size (98.9k voxels, the stem's 32 -> 32 K3 submanifold
    layer with the bench's HALVE | DENSITY_ORDER all-OS map): wgrad over every pair
    against the oracle, dgrad on 2048 sampled rows (the oracle's gather form)."""
    coords = synth.make_scan(2, 0)
    spec = _spec_for(coords)
    c = oracle.sort_coords(coords)[0]
    k = _keys(c, spec)
    km = spc.spc_build_kmap(k, k, spec, spc.Geom(3, 1, 1, 1, 0), -1, 1 | 8)
    F = synth.make_features(len(c), 32, seed=21)
    G = synth.make_features(len(c), 32, seed=22)
    W = synth.make_weights(27, 32, 32, seed=23, nnz_per_out=6)
    Fg, Gg = torch.from_numpy(F).to(DEV).bfloat16(), torch.from_numpy(G).to(DEV).bfloat16()
    dW = spc.spc_conv_wgrad(km, Fg, Gg, 32, 32)
    Wp = spc.spc_prepare_weight_ex(torch.from_numpy(W).to(DEV).bfloat16(), spc.SPC_WEIGHT_DGRAD_MIRROR)
    dF = spc.spc_conv_forward(km, Gg, Wp, 32, 32, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert _rel(dW.cpu().numpy().astype(np.float64), oracle.conv_wgrad(c, c, 3, 1, F, G)) <= 2e-3
    # 96 -> 96 on the all-WS halved map the network's backward uses: 32 KB stages, so a
    # ring of 6 stages for 8 producer warps (only 6 may run: the parity-skew limit)
    kw = spc.spc_build_kmap(k, k, spec, spc.Geom(3, 1, 1, 1, 0), 0, 1)
    F9 = synth.make_features(len(c), 96, seed=24)
    G9 = synth.make_features(len(c), 96, seed=25)
    dW9 = spc.spc_conv_wgrad(kw, torch.from_numpy(F9).to(DEV).bfloat16(), torch.from_numpy(G9).to(DEV).bfloat16(),
                             96, 96)
    torch.cuda.synchronize()
    assert _rel(dW9.cpu().numpy().astype(np.float64), oracle.conv_wgrad(c, c, 3, 1, F9, G9)) <= 2e-3
    rows = np.random.default_rng(0).choice(len(c), 2048, replace=False)
    ref = oracle.conv_dgrad_rows(c, c, rows, 3, 1, G, W)
    assert _rel(dF.cpu().numpy()[rows].astype(np.float64), ref) <= 2e-3


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_add_rows_and_inplace_residual_accumulation(dt):
    """spc_add_rows (the residual branch of a backward pass) on column slices with a live
    count, and spc_conv_forward with residual == output (gradient accumulation): every
    element read, then written, by one thread."""
    tdt = TDT[dt]
    rng = np.random.default_rng(1)
    A = torch.from_numpy(rng.uniform(-1, 1, (500, 48)).astype(np.float32)).to(DEV).to(tdt)
    B = torch.from_numpy(rng.uniform(-1, 1, (500, 40)).astype(np.float32)).to(DEV).to(tdt)
    ref = A.float().clone()
    n_dev = torch.tensor([300], dtype=torch.int64, device=DEV)
    spc.spc_add_rows(A[:, 8:40], B[:, 0:32], n_dev=n_dev)
    torch.cuda.synchronize()
    ref[:300, 8:40] = (ref[:300, 8:40] + B[:300, 0:32].float()).to(tdt).float()
    assert torch.equal(A.float(), ref)
    # the first contribution to a gradient overwrites (accumulate = 0)
    spc.spc_add_rows(A[:, 0:16], B[:, 16:32], n_dev=n_dev, accumulate=False)
    torch.cuda.synchronize()
    ref[:300, 0:16] = B[:300, 16:32].float()
    assert torch.equal(A.float(), ref)
    # in-place accumulation through the conv's residual operand (OS, WS and hybrid maps)
    spec, c, _ = _case(3000, seed=4)
    k = _keys(c, spec)
    for t, fl in ((-1, 8), (0, 1), (2, 1)):
        km = spc.spc_build_kmap(k, k, spec, spc.Geom(3, 1, 1, 1, 0), t, fl)
        F = synth.make_features(len(c), 32, seed=6, dtype=dt)
        W = synth.make_weights(27, 32, 32, seed=7, nnz_per_out=8, dtype=dt)
        G0 = synth.make_features(len(c), 32, seed=8, dtype=dt)
        G = torch.from_numpy(G0).to(DEV).to(tdt)
        spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).to(tdt), spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).to(tdt)),
                             32, 32, out=G, residual=G)
        torch.cuda.synchronize()
        ref = oracle.conv(c, c, 3, 1, F, W) + G0
        got = G.float().cpu().numpy().astype(np.float64)
        tol = 1e-5 if dt == "f32" else 2e-3
        ulp = 0 if dt == "f32" else np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        assert (np.abs(got - ref) <= ulp + tol * np.abs(ref).max()).all(), (t, fl)
