"""CTA pairs (cta_group::2, SPC_OPT_CONV_CTA_PAIR): the M = 256 MMAs of a pair, each CTA
holding 128 rows of a 256-row tile and half of every weight tile, against the oracle's
Eq. (2): OS (canonical and density-ordered), WS (halved), hybrid, strided, transposed,
C_out 192 / 256 / 384 (tiled), ragged tails and a pair whose second CTA has no rows."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _keys(c, spec):
    return torch.from_numpy(oracle.pack(c, spec.astuple())[0].view(np.int64)).to(DEV)


@pytest.fixture(autouse=True)
def _pairs():
    spc.spc_set_option(spc.SPC_OPT_CONV_CTA_PAIR, 2)
    yield
    spc.spc_set_option(spc.SPC_OPT_CONV_CTA_PAIR, -1)


@pytest.mark.parametrize("n_cut,kind,t,flags,c_in,c_out,res", [
    (6000, "subm", -1, 0, 64, 256, False), (6000, "subm", -1, 8, 128, 256, True), (6000, "subm", -1, 8, 256, 192, False),
    (100, "subm", -1, 0, 64, 256, False), (300, "subm", -1, 8, 64, 256, True), (6000, "subm", 0, 1, 64, 256, False),
    (6000, "subm", 2, 9, 256, 256, True), (6000, "subm", 0, 0, 32, 384, False), (6000, "strided", -1, 0, 64, 256, False),
    (6000, "transposed", 0, 0, 64, 256, False), (2000, "subm5", 3, 9, 64, 256, False)])
def test_cta_pair_conv(n_cut, kind, t, flags, c_in, c_out, res):
    coords = synth.make_scan(1, 0)[:n_cut]
    spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
    fine = oracle.sort_coords(coords)[0]
    coarse = oracle.downsample(fine, 2)
    K = 5 if kind == "subm5" else 3
    fk = _keys(fine, spec)
    if kind.startswith("subm"):
        ic, oc, ik, ok, g = fine, fine, fk, fk, spc.Geom(K, 1, 1, 1, 0)
    elif kind == "strided":
        ic, oc, ik, ok, g = fine, coarse, fk, _keys(coarse, spec), spc.Geom(3, 2, 1, 1, 0)
    else:
        ic, oc, ik, ok, g = coarse, fine, _keys(coarse, spec), fk, spc.Geom(3, 2, 1, 1, 1)
    km = spc.spc_build_kmap(ik, ok, spec, g, t, flags)
    F = synth.make_features(len(ic), c_in, seed=c_in)
    W = synth.make_weights(K ** 3, c_in, c_out, seed=c_out, nnz_per_out=10)
    R = synth.make_features(len(oc), c_out, seed=5) if res else None
    Wg = spc.spc_prepare_weight(torch.from_numpy(W).to(DEV).bfloat16())
    out = spc.spc_conv_forward(km, torch.from_numpy(F).to(DEV).bfloat16(), Wg, c_in, c_out,
                               out_dtype=torch.bfloat16 if res else torch.float32,
                               residual=None if R is None else torch.from_numpy(R).to(DEV).bfloat16())
    torch.cuda.synchronize()
    ref = oracle.conv(ic, oc, K, 1, F, W, transposed=(kind == "transposed"))
    got = out.float().cpu().numpy().astype(np.float64)
    if res:
        ref = ref + R.astype(np.float64)
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        assert (np.abs(got - ref) <= ulp + 1e-5 * np.abs(ref).max()).all()
    else:
        assert np.abs(got - ref).max() <= 2e-3 * np.abs(ref).max()
