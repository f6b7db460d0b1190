"""Voxelization front-end on the raw points of a BASELINE scan: device time
of spc_voxelize (captured in a CUDA graph, L2 flushed between replays, CUDA events), the
algorithmic bytes it must move, and the CPU oracle on the same points.  One JSON line.

  python scripts/voxelize_bench.py [--config 2] [--reps 50]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()

P, grid = synth.make_points(a.config, 0)
n = P.shape[0]
v = np.floor(P[:, :3] / np.asarray(grid, np.float32)).astype(np.int64)
spec = spc.spc_plan_pack(v.min(0), v.max(0), 1, 16, 16)
dev = torch.device("cuda")
Pt = torch.from_numpy(P).to(dev)            # rows (x, y, z, intensity): features = the whole row
s = torch.cuda.Stream(dev)
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        res = spc.spc_voxelize(Pt, grid, spec, feats=Pt, out_dtype=torch.bfloat16, stream=s)
torch.cuda.synchronize()
n_vox = int(res[1].item())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    res = spc.spc_voxelize(Pt, grid, spec, feats=Pt, out_dtype=torch.bfloat16, stream=s)
flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device=dev)
ts = []
for i in range(a.reps + 3):
    flush.fill_(i & 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
us = float(np.median(ts[3:]))
# algorithmic bytes: every point row read once (16 B), each voxel's key (8 B) and bf16 mean
# row (8 B) written once, the point -> voxel index (4 B) written once
alg = n * 16 + n_vox * (8 + 8) + n * 4
peaks = {}
try:
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
except Exception:
    pass
hbm = float(peaks.get("hbm_gbs", peaks.get("copy_gbs", 6544.0)) or 6544.0)
import oracle  # noqa: E402  (CPU baseline only)
t0 = time.perf_counter()
oc, _, _ = oracle.voxelize(P[:, :3], grid, feats=P)
cpu_s = time.perf_counter() - t0
assert len(oc) == n_vox
print(json.dumps({"what": "spc_voxelize (quantise + pack + sort + unique + mean, bf16 out)", "config": a.config,
                  "n_points": n, "n_voxels": n_vox, "grid": grid, "us": round(us, 2),
                  "mpoints_per_s": round(n / us, 1), "algorithmic_bytes": alg,
                  "algorithmic_gbs": round(alg / (us * 1e-6) / 1e9, 1), "hbm_peak_gbs": hbm,
                  "frac": round(alg / (us * 1e-6) / 1e9 / hbm, 4),
                  "cpu_oracle_s": round(cpu_s, 3), "cpu_oracle_threads": 1,
                  "l2": "flushed (320 MB write) between replays", "cuda_graph": True}))
