"""Network-wide kernel-map build (A13) of the whole C4 batch on ONE GPU: HBM-roofline evidence.

8 Waymo-shaped scans (~1.63M voxels) packed with a batch field, MinkUNet-42's 5 levels and 18
distinct maps built by spc_network_kmaps.  The maps (~0.4 GB) exceed the 126 MB L2, and L2
is flushed (320 MB write) before every repetition, so this is the configuration where the
kernel-map build is HBM-bound.

Algorithmic bytes: per level m: read 8 B per V_0 key, write 8 B per unique
output; per map: 8 N_in + 8 N_out (keys) + 4 N_out K_dense (OS table) + 8 nnz_ws (WS pairs as
stored, halved for submanifold) + 4 K^3 (counts).

python scripts/kmap_c4.py [--reps 20] [--t default|os] [--no-order]    (prints one JSON line)
Under ncu:  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
              -k regex:k_kmap python scripts/kmap_c4.py --reps 1
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_20834_b200 as spc  # noqa: E402
from paper_2511_20834_b200.network import SparseUNet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--t", default="default", choices=["default", "os", "ws"])
ap.add_argument("--no-order", action="store_true", help="build without SPC_KMAP_DENSITY_ORDER")
a = ap.parse_args()

import bench  # noqa: E402  (the same C4 workload bench.py --config 4 times)

coords_np, _, _, _ = bench.workload(0, 4, 1)
n = coords_np.shape[0]
spec = spc.spc_plan_pack(coords_np[:, 1:].min(0), coords_np[:, 1:].max(0), 8, 16, 16)
net = SparseUNet(n, spec, density_order=not a.no_order)
if a.t != "default":
    net.set_t({mk: (spc.SPC_T_ALL_OS if a.t == "os" else 0) for mk in net.map_keys if mk[0] > 1})
coords = torch.from_numpy(coords_np).cuda()
spc.spc_pack_sort(coords, spec, status=net.status, keys_out=net.keys, perm_out=net.perm, ws=net.sort_ws)
net.index()
torch.cuda.synchronize()

level_n = [n] + [int(v) for v in net.level_n.cpu().tolist()[1:]]
alg = 0
# levels 1..4: each reads the V_0 keys (Eq. 3) and writes its unique keys
for m in range(1, net.n_levels):
    alg += 8 * n + 8 * level_n[m]
per_map = []
for mk, km in net.maps.items():
    K, s, ts, tr = mk
    lv = int(round(np.log2(ts)))
    if tr:
        lin, lout = lv + 1, lv
    elif s == 2:
        lin, lout = lv, lv + 1
    else:
        lin = lout = lv
    n_in, n_out = level_n[lin], level_n[lout]
    cnt = km.counts().cpu().numpy()
    nnz_ws = int(cnt[spc.SPC_MAX_KVOL:spc.SPC_MAX_KVOL + km.n_lists].sum())
    b = 8 * n_in + 8 * n_out + 4 * n_out * km.k_dense + 8 * nnz_ws + 4 * K ** 3
    per_map.append({"map": list(mk), "n_in": n_in, "n_out": n_out, "k_dense": km.k_dense, "nnz_ws": nnz_ws,
                    "bytes": b})
    alg += b

flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device="cuda")
ms = []
for r in range(a.reps + 2):
    flush.fill_(r & 0xFF)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    net.index()
    e1.record()
    torch.cuda.synchronize()
    if r >= 2:
        ms.append(e0.elapsed_time(e1))
t = float(np.median(ms)) / 1e3
peaks = bench.measured_peaks()
peak = peaks.get("hbm_gbs", 6650.0)
print(json.dumps({"what": "C4 batch network-wide kernel maps on one GPU (levels + 18 maps)", "n_voxels": n,
                  "levels": level_n, "t": a.t, "density_order": not a.no_order, "median_us": t * 1e6,
                  "algorithmic_bytes": alg, "achieved_gbs": alg / t / 1e9, "peak_gbs": peak,
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s",
                  "frac": alg / t / 1e9 / peak, "maps": per_map}))
