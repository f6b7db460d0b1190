"""Randomised acceptance suite (the SPEC acceptance items (1), (2), (4), (7)):
200 seeded instances -- n in {10, 1k, 10k}, K in {1, 3, 5}, layer stride 1/2 (strided or
transposed), dilation 1/2, random dataflow threshold t, halving and density order, 1-3
batches, random or surface clouds, channels 16/32 (bf16) and 8/16 (fp32) -- each built and
convolved through the C ABI and compared with the oracle: the z-delta map equals the hash
map as a set of triples (the oracle's map is pinned to brute force), an all-OS map built by
the paper's Simple BSearch equals it too, and the features equal Eq. (2)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"
N_CASES = 200


def _case(i):
    rng = np.random.default_rng(20834 + i)
    n = int(rng.choice([10, 1000, 10000], p=[0.3, 0.45, 0.25]))
    K = int(rng.choice([1, 3, 5], p=[0.15, 0.6, 0.25]))
    kind = str(rng.choice(["subm", "strided", "transposed"], p=[0.6, 0.2, 0.2])) if K > 1 else "subm"
    d = int(rng.choice([1, 2], p=[0.8, 0.2])) if kind == "subm" else 1
    nb = int(rng.integers(1, 4))
    if rng.uniform() < 0.5:
        c = synth.random_cloud(n, max(4, int(round((n / nb) ** (1 / 3) * 2.2))), seed=i, n_batch=nb)
    else:
        c = synth.surface_cloud(n, seed=i, n_batch=nb)[:n]
    l1max = 3 * (K - 1) // 2
    t = int(rng.integers(-1, l1max + 2))
    flags = 0
    if kind == "subm" and rng.uniform() < 0.5:
        flags |= spc.SPC_KMAP_HALVE_SYMMETRIC
    if rng.uniform() < 0.5:
        flags |= spc.SPC_KMAP_DENSITY_ORDER
    f32 = rng.uniform() < 0.2
    ci, co = (int(rng.choice([8, 16])), int(rng.choice([8, 16]))) if f32 else \
        (int(rng.choice([16, 32])), int(rng.choice([16, 32])))
    return dict(c=c, K=K, kind=kind, d=d, t=t, flags=flags, f32=f32, ci=ci, co=co, seed=i)


def _keys(c_sorted, spec):
    k, bad = oracle.pack(c_sorted, spec.astuple())
    assert bad == 0
    return torch.from_numpy(k.view(np.int64)).to(DEV)


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_instance(i):
    p = _case(i)
    c = oracle.sort_coords(p["c"])[0]
    K, kind, d = p["K"], p["kind"], p["d"]
    spec = spc.spc_plan_pack(c[:, 1:].min(0), c[:, 1:].max(0), int(c[:, 0].max()) + 1, 16, 16)
    fine = c
    coarse = oracle.downsample(c, 2)
    if kind == "subm":
        a, b, g, tr = fine, fine, spc.Geom(K, 1, d, 1, 0), False
    elif kind == "strided":
        a, b, g, tr = fine, coarse, spc.Geom(K, 2, 1, 1, 0), False
    else:
        a, b, g, tr = coarse, fine, spc.Geom(K, 2, 1, 1, 1), True
    ka = _keys(a, spec)
    kb = ka if a is b else _keys(b, spec)
    km = spc.spc_build_kmap(ka, kb, spec, g, p["t"], p["flags"])
    ref_map = oracle.kmap(a, b, K, d, transposed=tr)
    assert np.array_equal(spc.spc_kmap_export(km), ref_map), p
    # the paper's Simple BSearch baseline (all-OS maps only) builds the same map
    if not tr and d == 1:
        kbs = spc.spc_build_kmap(ka, kb, spec, g, spc.SPC_T_ALL_OS, spc.SPC_KMAP_SIMPLE_BSEARCH)
        assert np.array_equal(spc.spc_kmap_export(kbs), ref_map)
    dt = "f32" if p["f32"] else "bf16"
    tdt = torch.float32 if p["f32"] else torch.bfloat16
    F = synth.make_features(len(a), p["ci"], seed=p["seed"], dtype=dt)
    W = synth.make_weights(K ** 3, p["ci"], p["co"], seed=p["seed"] + 1, nnz_per_out=6, dtype=dt)
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).to(tdt),
                               spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).to(tdt)), p["ci"], p["co"],
                               out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle.conv(a, b, K, d, F, W, transposed=tr)
    m = np.abs(ref).max()
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref).max() / (m if m > 0 else 1.0)
    assert err <= (1e-5 if p["f32"] else 2e-3), (p, err)


def test_density_ratio_on_surfaces():
    """SPEC acceptance (4) / P:207-208: on LiDAR-like surfaces the offsets adjacent to the
    centre (L1 = 1) match at least 3x as often as the corners (L1 = L1max)."""
    c = oracle.sort_coords(synth.make_scan(1, 0))[0]
    spec = spc.spc_plan_pack(c[:, 1:].min(0), c[:, 1:].max(0), 1, 16, 16)
    k = _keys(c, spec)
    km = spc.spc_build_kmap(k, k, spec, spc.Geom(3, 1, 1, 1, 0), -1, 0)
    cnt = km.counts().cpu().numpy()[:27].astype(np.float64)
    off = np.array([(x, y, z) for x in (-1, 0, 1) for y in (-1, 0, 1) for z in (-1, 0, 1)])
    l1 = np.abs(off).sum(1)
    assert cnt[l1 == 1].mean() >= 3 * cnt[l1 == 3].mean()
