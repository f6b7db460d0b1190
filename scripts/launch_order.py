"""Device-side kernel durations of one MinkUNet-42 forward (C2), in launch order, grouped by
layer (torch.profiler / CUPTI; kernel times are device-side, independent of Python overhead).

python scripts/launch_order.py [--config 2] [--graph]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--no-tune", action="store_true")
a = ap.parse_args()

coords_np = synth.make_scan(a.config, 0)
spec = bench.spec_for(coords_np)
net = SparseNet(coords_np.shape[0], spec, net="secondk5" if a.config == 3 else "minkunet42")
coords = torch.from_numpy(coords_np).cuda()
feats = torch.zeros(coords.shape[0], C_IN_PAD, dtype=torch.bfloat16, device="cuda")
feats[:, :4] = torch.randn(coords.shape[0], 4, device="cuda").bfloat16()
stream = torch.cuda.current_stream()
if not a.no_tune:
    print("t:", bench.tune(net, coords, feats, stream), file=sys.stderr)
for _ in range(3):
    net.forward(coords, feats)
torch.cuda.synchronize()

marker = torch.zeros(1, device="cuda")
names = [s.name for s in net.layers]
import paper_2511_20834_b200 as spc  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    spc.spc_pack_sort(coords, net.spec, status=net.status, keys_out=net.keys, perm_out=net.perm, ws=net.sort_ws)
    spc.spc_gather_rows(feats, net.perm, out=net.bufs["x0"])
    net.index()
    for i in range(len(names)):
        marker.add_(1)          # separator kernel
        net.conv(i)
    marker.add_(1)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if "CUDA" in str(getattr(e, "device_type", ""))]
ev.sort(key=lambda e: e.time_range.start)
li = -1
rows = []
prev_end = None
for e in ev:
    nm = e.name.split("(")[0].replace("void ", "")
    if "elementwise" in nm:
        li += 1
        continue
    gap = 0.0 if prev_end is None else e.time_range.start - prev_end
    rows.append(("index" if li < 0 else names[li] if li < len(names) else "-", nm[:40], e.time_range.elapsed_us(), gap))
    prev_end = e.time_range.end
print(f"{'layer':22s} {'kernel':40s} {'us':>8s}")
per = {}
for r in rows:
    print(f"{r[0]:22s} {r[1]:40s} {r[2]:8.1f}")
    per[r[0]] = per.get(r[0], 0.0) + r[2]
print()
for k, v in per.items():
    print(f"{k:22s} {v:8.1f}")
print(f"kernels {len(rows)}  busy {sum(per.values()):.1f} us  conv {sum(v for k, v in per.items() if k != 'index'):.1f} us")
