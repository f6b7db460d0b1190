"""NEXT-1: 32-bit single-scan keys (P:315 packs one scan into 32 bits, 12/12/8; the
paper's layer-wise results use 32-bit packing).  spc_pack_sort32 and
spc_build_kmap32 against the oracle: keys and permutation bit-exact, kernel maps
bit-exact as triple sets (the same maps as the 64-bit path), features within tolerance."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _spec(coords, stride=16, reach=16):
    return spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, stride, reach)


def _keys32(c, spec):
    k, bad = oracle.pack(c, spec.astuple())
    assert bad == 0 and int(k.max()) < 2 ** 32
    return torch.from_numpy(k.astype(np.uint32).view(np.int32)).to(DEV)


@pytest.mark.parametrize("config", [1, 2])
def test_pack_sort32_bit_exact(config):
    coords = synth.make_scan(config, 0)
    spec = _spec(coords)
    assert spec.used_bits() <= 32, spec
    keys, perm, status = spc.spc_pack_sort(torch.from_numpy(coords).to(DEV), spec, key_bits=32)
    torch.cuda.synchronize()
    assert keys.dtype == torch.int32 and int(status.item()) == 0
    s, p, _ = oracle.sort_coords(coords)
    ref, _ = oracle.pack(s, spec.astuple())
    np.testing.assert_array_equal(keys.cpu().numpy().view(np.uint32).astype(np.uint64), ref)
    np.testing.assert_array_equal(perm.cpu().numpy(), p)
    # the 64-bit path sorts to the same order
    k64, p64, _ = spc.spc_pack_sort(torch.from_numpy(coords).to(DEV), spec)
    np.testing.assert_array_equal(p64.cpu().numpy(), p)


def test_pack_sort32_flags_and_width_check():
    coords = synth.make_scan(1, 0)
    spec = _spec(coords)
    dup = np.concatenate([coords, coords[:3]])
    _, _, st = spc.spc_pack_sort(torch.from_numpy(dup).to(DEV), spec, key_bits=32)
    torch.cuda.synchronize()
    assert int(st.item()) & spc.SPC_FLAG_DUPLICATE
    wide = spc.spc_plan_pack((-40000, -40000, -500), (40000, 40000, 500), 1, 16, 16)   # > 32 bits
    assert wide.used_bits() > 32
    with pytest.raises(spc.SpcError):
        spc.spc_pack_sort(torch.from_numpy(coords).to(DEV), wide, key_bits=32)


MAP_CASES = [(3, 1, "subm", -1, 0), (3, 1, "subm", 2, 1), (3, 1, "subm", 0, 1), (3, 1, "subm", -1, 8),
             (5, 1, "subm", 3, 9), (3, 2, "subm", 2, 1), (3, 1, "strided", -1, 8), (3, 1, "strided", 0, 0),
             (3, 1, "transposed", -1, 8), (5, 1, "transposed", 2, 0)]


@pytest.mark.parametrize("K,d,kind,t,flags", MAP_CASES)
def test_kmap32_bit_exact(K, d, kind, t, flags):
    coords = synth.make_scan(1, 1)
    spec = _spec(coords)
    fine = oracle.sort_coords(coords)[0]
    coarse = oracle.downsample(fine, 2)
    fk = _keys32(fine, spec)
    if kind == "subm":
        ik, ok, ic, oc, g = fk, fk, fine, fine, spc.Geom(K, 1, d, 1, 0)
    elif kind == "strided":
        ik, ok, ic, oc, g = fk, _keys32(coarse, spec), fine, coarse, spc.Geom(K, 2, d, 1, 0)
    else:
        ik, ok, ic, oc, g = _keys32(coarse, spec), fk, coarse, fine, spc.Geom(K, 2, d, 1, 1)
    km = spc.spc_build_kmap(ik, ok, spec, g, t, flags | spc.SPC_KMAP_COUNT_SEARCHES)
    assert km.c.key_bits == 32
    ref = oracle.kmap(ic, oc, K, d, transposed=(kind == "transposed"))
    np.testing.assert_array_equal(spc.spc_kmap_export(km), ref)
    if kind == "subm" and not (flags & 1):
        assert km.search_stats().cpu().numpy()[0] == len(oc) * K * K
    # same map as the 64-bit build
    k64 = lambda x: torch.from_numpy(oracle.pack(x, spec.astuple())[0].view(np.int64)).to(DEV)
    i64 = k64(ic)
    o64 = i64 if oc is ic else k64(oc)
    km64 = spc.spc_build_kmap(i64, o64, spec, g, t, flags)
    np.testing.assert_array_equal(spc.spc_kmap_export(km64), ref)


def test_conv_on_kmap32():
    coords = synth.make_scan(1, 0)[:6000]
    spec = _spec(coords)
    c = oracle.sort_coords(coords)[0]
    fk = _keys32(c, spec)
    km = spc.spc_build_kmap(fk, fk, spec, spc.Geom(3, 1, 1, 1, 0), 2, spc.SPC_KMAP_HALVE_SYMMETRIC | 8)
    F = synth.make_features(len(c), 32, seed=3)
    W = synth.make_weights(27, 32, 64, seed=4, nnz_per_out=10)
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(),
                               spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16()), 32, 64,
                               out_dtype=torch.float32)
    ref = oracle.conv(c, c, 3, 1, F, W)
    got = out.cpu().numpy().astype(np.float64)
    assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max()
