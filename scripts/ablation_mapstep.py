"""NEXT-1 ablation on B200 (Fig. mapstep): kernel-map build time of the one-shot
z-delta search (|V_q| K^2 binary searches + cursor) against the paper's Simple BSearch
baseline (|V_q| K^3 independent binary searches), same all-OS layout, same maps (both are
parity-tested against the oracle).  Device time = sum of the build's kernel durations
(torch profiler), median over reps.  Prints one JSON line per (scene, K).

python scripts/ablation_mapstep.py [--reps 5]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import bench
import paper_2511_20834_b200 as spc

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()


def kernel_us(fn):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return sum(e.device_time_total for e in prof.key_averages())


for cfg, label in ((2, "C2 KITTI-like scan"), (4, "C4 batch of 8 Waymo-like scans")):
    coords_np, _, _, _ = bench.workload(0, cfg, 1)
    nb = int(coords_np[:, 0].max()) + 1
    spec = spc.spc_plan_pack(coords_np[:, 1:].min(0), coords_np[:, 1:].max(0), nb, 16, 16)
    keys, _, _ = spc.spc_pack_sort(torch.from_numpy(coords_np).cuda(), spec)
    n = keys.shape[0]
    for K in (3, 5):
        g = spc.Geom(K, 1, 1, 1, 0)
        res = {}
        for name, fl in (("zdelta", 0), ("simple_bsearch", spc.SPC_KMAP_SIMPLE_BSEARCH)):
            spc.spc_build_kmap(keys, keys, spec, g, -1, fl)   # warm-up
            ts = [kernel_us(lambda: spc.spc_build_kmap(keys, keys, spec, g, -1, fl)) for _ in range(a.reps)]
            res[name] = float(np.median(ts))
        print(json.dumps({"what": "kernel-map build (all-OS submanifold map), device us", "scene": label,
                          "n_voxels": int(n), "K": K, "searches_zdelta": int(n) * K * K,
                          "searches_simple_bsearch": int(n) * K ** 3, "zdelta_us": round(res["zdelta"], 1),
                          "simple_bsearch_us": round(res["simple_bsearch"], 1),
                          "speedup": round(res["simple_bsearch"] / res["zdelta"], 2)}), flush=True)
