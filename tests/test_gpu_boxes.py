"""SURVEY NEXT-3 on the GPU: kernel maps and Eq. (2) over (Kx, Ky, Kz) offset boxes with
even sizes {0..K-1} (reading E1: the K = 2 stride-2 down / up layers, non-cubic (3, 1, 1)
kernels), and spconv's regular output rule -- bit-exact maps and output sites against
the oracle (oracle.kmap / oracle.regular_outputs over the same boxes), features within
the bf16 bound of test_gpu_parity."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _setup(scan=1, n=None):
    coords = synth.make_scan(1, scan)
    if n:
        coords = coords[:n]
    spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
    fine = oracle.sort_coords(coords)[0]
    coarse = oracle.downsample(fine, 2)
    fk = torch.from_numpy(oracle.pack(fine, spec.astuple())[0].view(np.int64)).to(DEV)
    ck = torch.from_numpy(oracle.pack(coarse, spec.astuple())[0].view(np.int64)).to(DEV)
    return spec, fine, coarse, fk, ck


BOX_MAPS = [
    # (box, kind, t, flags, dilation)
    ((2, 2, 2), "strided", -1, 0, 1), ((2, 2, 2), "strided", 0, 0, 1), ((2, 2, 2), "strided", 2, 8, 1),
    ((2, 2, 2), "transposed", -1, 0, 1), ((2, 2, 2), "transposed", 1, 0, 1),
    ((3, 1, 1), "subm", -1, 0, 1), ((3, 1, 1), "subm", 0, 1, 1), ((1, 3, 1), "subm", 1, 9, 1),
    ((1, 1, 3), "subm", -1, 8, 2), ((3, 3, 1), "strided", 2, 0, 1), ((4, 2, 3), "subm", -1, 0, 1),
    ((4, 2, 3), "subm", 2, 1, 1), ((5, 1, 3), "subm", 3, 9, 2), ((2, 4, 1), "transposed", 0, 0, 1),
]


def _geom_io(box, kind, d, fine, coarse, fk, ck):
    if kind == "subm":
        return spc.Geom(box, 1, d, 1, 0), fk, fk, fine, fine, False
    if kind == "strided":
        return spc.Geom(box, 2, d, 1, 0), fk, ck, fine, coarse, False
    return spc.Geom(box, 2, d, 1, 1), ck, fk, coarse, fine, True


@pytest.mark.parametrize("box,kind,t,flags,d", BOX_MAPS)
def test_box_kmap_bit_exact(box, kind, t, flags, d):
    spec, fine, coarse, fk, ck = _setup()
    g, ik, ok, ic, oc, tr = _geom_io(box, kind, d, fine, coarse, fk, ck)
    km = spc.spc_build_kmap(ik, ok, spec, g, t, flags)
    np.testing.assert_array_equal(spc.spc_kmap_export(km), oracle.kmap(ic, oc, box, d, transposed=tr))


@pytest.mark.parametrize("box,kind,t,flags,c_in,c_out", [
    ((2, 2, 2), "strided", -1, 0, 32, 64), ((2, 2, 2), "strided", 0, 0, 64, 64), ((2, 2, 2), "transposed", -1, 8, 64, 32),
    ((2, 2, 2), "transposed", 0, 0, 128, 96), ((3, 1, 1), "subm", 1, 1, 32, 32), ((4, 2, 3), "subm", -1, 8, 16, 48),
    ((4, 2, 3), "subm", 2, 0, 96, 128), ((1, 3, 1), "subm", 0, 1, 256, 256)])
def test_box_conv_matches_eq2(box, kind, t, flags, c_in, c_out):
    spec, fine, coarse, fk, ck = _setup(0, 6000)
    g, ik, ok, ic, oc, tr = _geom_io(box, kind, 1, fine, coarse, fk, ck)
    km = spc.spc_build_kmap(ik, ok, spec, g, t, flags)
    F = synth.make_features(len(ic), c_in, seed=c_in)
    W = synth.make_weights(g.k_vol(), c_in, c_out, seed=c_out, nnz_per_out=4)
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(), Wg, c_in, c_out, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle.conv(ic, oc, box, 1, F, W, transposed=tr)
    got = out.cpu().numpy().astype(np.float64)
    assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max()


@pytest.mark.parametrize("box,s,d", [(3, 2, 1), ((3, 1, 1), 2, 1), (5, 2, 1), (3, 1, 1), ((2, 2, 2), 2, 1), (3, 2, 2)])
def test_regular_outputs_bit_exact(box, s, d):
    spec, fine, coarse, fk, ck = _setup()
    g = spc.Geom(box, s, d, 1, 0)
    keys, n_out = spc.spc_regular_outputs(fk, spec, g)
    torch.cuda.synchronize()
    ref = oracle.regular_outputs(fine, box, d, s)
    m = int(n_out.item())
    assert m == len(ref)
    np.testing.assert_array_equal(keys[:m].cpu().numpy(), oracle.pack(ref, spec.astuple())[0].view(np.int64))
    if box == (2, 2, 2) and s == 2:
        np.testing.assert_array_equal(ref, coarse)     # K = 2, s = 2: Eq. (1)'s V_q


def test_regular_conv_end_to_end():
    """A spconv-style SparseConv3d (K = 3, stride 2, padding 1): regular output sites, the
    map onto them and Eq. (2), each checked against the oracle."""
    spec, fine, coarse, fk, ck = _setup(0)
    g = spc.Geom(3, 2, 1, 1, 0)
    keys, n_out = spc.spc_regular_outputs(fk, spec, g)
    m = int(n_out.item())
    ok = keys[:m].contiguous()
    reg = oracle.regular_outputs(fine, 3, 1, 2)
    km = spc.spc_build_kmap(fk, ok, spec, g, -1, 8)
    np.testing.assert_array_equal(spc.spc_kmap_export(km), oracle.kmap(fine, reg, 3, 1))
    F = synth.make_features(len(fine), 32, seed=1)
    W = synth.make_weights(27, 32, 64, seed=2, nnz_per_out=4)
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(), Wg, 32, 64, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle.conv(fine, reg, 3, 1, F, W)
    assert np.abs(out.cpu().numpy() - ref).max() <= 2e-3 * np.abs(ref).max()
    assert m > len(coarse)   # the regular rule dilates Eq. (1)'s sites
