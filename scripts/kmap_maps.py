"""Per-map standalone kernel-map build times on the C4 batch (which maps dominate k_kmap_zdelta).

python scripts/kmap_maps.py [--config 4]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2511_20834_b200 as spc
from paper_2511_20834_b200.network import SparseUNet

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
a = ap.parse_args()
coords_np, _, _, _ = bench.workload(0, a.config, 1)
n = coords_np.shape[0]
spec = spc.spc_plan_pack(coords_np[:, 1:].min(0), coords_np[:, 1:].max(0), 8, 16, 16)
net = SparseUNet(n, spec)
coords = torch.from_numpy(coords_np).cuda()
spc.spc_pack_sort(coords, spec, status=net.status, keys_out=net.keys, perm_out=net.perm, ws=net.sort_ws)
net.index()
torch.cuda.synchronize()
ln = [n] + [int(v) for v in net.level_n.cpu().tolist()[1:]]
lk = [net.keys] + [net.level_keys[l, :ln[l]] for l in range(1, len(ln))]
tot = 0
for mk in net.map_keys:
    K, s, ts, tr = mk
    lv = int(round(np.log2(ts)))
    lin, lout = (lv + 1, lv) if tr else ((lv, lv + 1) if s == 2 else (lv, lv))
    t = net.t[mk]
    fl = spc.SPC_KMAP_HALVE_SYMMETRIC if (s == 1 and K > 1) else 0
    g = spc.Geom(K, s, 1, ts, tr)
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        km = spc.spc_build_kmap(lk[lin], lk[lout], spec, g, t, fl)
        e1.record()
        torch.cuda.synchronize()
        if rep == 1:
            ms = []
        if rep >= 1:
            ms.append(e0.elapsed_time(e1))
    us = float(np.median(ms)) * 1e3
    tot += us
    print(f"map {str(mk):18s} t={t:3d} n_in {ln[lin]:8d} n_out {ln[lout]:8d} k_dense {km.k_dense:3d} lists {km.n_lists:3d}: "
          f"{us:8.1f} us  {us / (ln[lout] / 128):6.3f} us/tile", flush=True)
print(f"total {tot:.1f} us")
