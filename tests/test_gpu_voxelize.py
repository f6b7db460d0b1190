"""GPU parity of the voxelization front-end (P:96 v = floor(p/g), S:70-78,
S:132) against oracle.voxelize: voxel keys, voxel count and the point -> voxel map
bit-exact; mean features within the fp32 summation bound derived below."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc

pytestmark = pytest.mark.gpu
DEV = "cuda"
U32 = 2.0 ** -24   # fp32 unit roundoff


def _spec_for_points(P, grid, n_batch=1):
    v = np.floor(P[:, :3] / np.asarray(grid, np.float32)).astype(np.int64)
    return spc.spc_plan_pack(v.min(0), v.max(0), n_batch, 16, 16)


def _check(P, grid, feats=None, batch=None, out_dtype=torch.float32, n_live=None):
    n_cap = P.shape[0]
    n = n_cap if n_live is None else n_live
    spec = _spec_for_points(P[:n], grid, 1 if batch is None else int(batch[:n].max()) + 1)
    Pt = torch.from_numpy(P).to(DEV)
    bt = None if batch is None else torch.from_numpy(batch).to(DEV)
    Ft = None if feats is None else torch.from_numpy(feats).to(DEV)
    n_dev = None if n_live is None else torch.tensor([n_live], dtype=torch.int64, device=DEV)
    keys, n_vox, pv, out, status, bad = spc.spc_voxelize(Pt, grid, spec, batch=bt, feats=Ft, out_dtype=out_dtype,
                                                         n_dev=n_dev)
    torch.cuda.synchronize()
    assert int(status.item()) == 0 and int(bad.item()) == -1
    c_ref, pv_ref, m_ref = oracle.voxelize(P[:n], grid, batch=None if batch is None else batch[:n],
                                           feats=None if feats is None else feats[:n])
    nv = int(n_vox.item())
    assert nv == len(c_ref)
    k_ref, nbad = oracle.pack(c_ref, spec.astuple())
    assert nbad == 0
    assert np.array_equal(keys[:nv].cpu().numpy(), k_ref.view(np.int64))
    assert np.array_equal(pv[:n].cpu().numpy(), pv_ref)
    if feats is not None:
        # fp32 sequential sum of m terms: |err| <= (m-1) u sum|f| (+ second order), the
        # division adds u |mean|, the output rounding half an ulp of its format
        cnt = np.bincount(pv_ref, minlength=nv).astype(np.float64)
        absum = np.stack([np.bincount(pv_ref, weights=np.abs(feats[:n, ch].astype(np.float64)), minlength=nv)
                          for ch in range(feats.shape[1])], 1)
        got = out[:nv].float().cpu().numpy().astype(np.float64)
        mant = 23 if out_dtype == torch.float32 else 7
        half_ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(m_ref), 1e-30))) - mant - 1)
        tol = 1.01 * ((cnt - 1)[:, None] * U32 * absum / cnt[:, None] + U32 * np.abs(m_ref)) + half_ulp + 1e-38
        assert (np.abs(got - m_ref) <= tol).all()
    return nv


def test_voxelize_random_cloud_batched():
    rng = np.random.default_rng(3)
    P = rng.uniform(-5, 5, (3000, 3)).astype(np.float32)
    P[::5] = P[7]                                     # merged voxels
    b = rng.integers(0, 3, 3000).astype(np.int32)
    F = rng.uniform(-1, 1, (3000, 5)).astype(np.float32)
    _check(P, (0.1, 0.1, 0.1), feats=F, batch=b)


@pytest.mark.parametrize("config,c,dt", [(1, 1, torch.float32), (1, 37, torch.bfloat16), (2, 4, torch.bfloat16)])
def test_voxelize_lidar_scan_full_size(config, c, dt):
    """Raw points of the C1 / C2 scans (125k / ~190k points): intensity only, a ragged 37
    channels, or (x, y, z, intensity) into bf16 -- the network's input layout."""
    P, grid = synth.make_points(config, 0)
    if c == 1:
        F = np.ascontiguousarray(P[:, 3:4])
    elif c == 4:
        F = np.ascontiguousarray(P[:, :4])
    else:
        F = np.random.default_rng(c).uniform(-1, 1, (P.shape[0], c)).astype(np.float32)
    nv = _check(np.ascontiguousarray(P[:, :3]), grid, feats=F, out_dtype=dt)
    assert nv > 10_000


def test_voxelize_edge_cases():
    # one point; every point in one voxel (long fp32 sums); points on grid planes
    _check(np.array([[0.3, -0.2, 7.0]], np.float32), (0.5, 0.5, 0.5), feats=np.array([[2.5]], np.float32))
    rng = np.random.default_rng(5)
    P = rng.uniform(0.0, 0.099, (4000, 3)).astype(np.float32)
    assert _check(P, (0.1, 0.1, 0.1), feats=rng.uniform(-1, 1, (4000, 3)).astype(np.float32)) == 1
    k = rng.integers(-40, 40, (2000, 3)).astype(np.float32) * np.float32(0.25)
    _check(k, (0.25, 0.25, 0.25), feats=rng.uniform(-1, 1, (2000, 2)).astype(np.float32))


def test_voxelize_device_count_and_empty():
    rng = np.random.default_rng(9)
    P = rng.uniform(-3, 3, (5000, 3)).astype(np.float32)
    F = rng.uniform(-1, 1, (5000, 8)).astype(np.float32)
    _check(P, (0.2, 0.2, 0.2), feats=F, n_live=3111)
    spec = spc.spc_plan_pack((0, 0, 0), (1, 1, 1), 1, 1, 0)
    keys, n_vox, pv, out, status, bad = spc.spc_voxelize(torch.zeros(0, 3, device=DEV), (1, 1, 1), spec)
    torch.cuda.synchronize()
    assert int(n_vox.item()) == 0 and int(bad.item()) == -1 and int(status.item()) == 0


def test_voxelize_flags_non_finite_and_range():
    """non-finite points are reported (flag + the first bad point index); a voxel
    outside the planned fields sets SPC_FLAG_RANGE (no silent truncation)."""
    rng = np.random.default_rng(2)
    P = rng.uniform(-2, 2, (1000, 3)).astype(np.float32)
    spec = _spec_for_points(P, (0.1, 0.1, 0.1))
    P[456, 2] = np.inf
    P[123, 0] = np.nan
    _, _, _, _, status, bad = spc.spc_voxelize(torch.from_numpy(P).to(DEV), (0.1, 0.1, 0.1), spec)
    torch.cuda.synchronize()
    assert int(status.item()) & 0x10 and int(bad.item()) == 123
    P = rng.uniform(-2, 2, (1000, 3)).astype(np.float32)
    spec = _spec_for_points(P, (0.1, 0.1, 0.1))
    P[17, 1] = 1e4                                      # far outside the planned field
    _, _, _, _, status, bad = spc.spc_voxelize(torch.from_numpy(P).to(DEV), (0.1, 0.1, 0.1), spec)
    torch.cuda.synchronize()
    assert int(status.item()) & 0x1 and int(bad.item()) == -1
