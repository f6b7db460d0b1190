"""Device timeline of one C2 step (spc_set_trace): per feature-kernel launch, when its
first CTA entered, when the PDL wait released, when the first tile record / first full
stage appeared, and when the median / last CTA left.  Runs the bench's configuration
(tuned t, HALVE | DENSITY_ORDER) as a captured CUDA graph and traces the last replay.

  python scripts/timeline.py [--config 2] [--t-from profiles/r2_tuned_t_c2.json] [--eager]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402
from paper_2511_20834_b200 import build as spc_build  # noqa: E402

# per-tile events are compiled only into the tracing build of the library
spc.LIB_PATH = spc_build.build(exp="trace", defines=["-DSPC_TRACE_TILES"])
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--t-from", default=os.path.join(bench.ROOT, "profiles", "r2_tuned_t_c2.json"))
ap.add_argument("--eager", action="store_true")
ap.add_argument("--out", default=None)
a = ap.parse_args()

coords_np, feats_np, _, net_name = bench.workload(0, a.config, 1)
n = coords_np.shape[0]
spec = bench.spec_for(coords_np)
dev = torch.device("cuda")
net = SparseNet(n, spec, device=dev, net=net_name)
if a.t_from and os.path.exists(a.t_from):
    net.set_t(bench.load_t(a.t_from))
coords = torch.from_numpy(coords_np).to(dev)
feats = torch.zeros(n, C_IN_PAD, dtype=torch.bfloat16, device=dev)
feats[:, :feats_np.shape[1]] = torch.from_numpy(feats_np).to(dev, torch.bfloat16)
buf = torch.zeros(1 + 2 * 400_000, dtype=torch.int64, device=dev)
net.forward(coords, feats)
torch.cuda.synchronize()
spc.spc_set_trace(buf)
s2 = torch.cuda.Stream(dev)
if a.eager:
    for _ in range(3):
        buf[0] = 0
        spc.spc_set_trace(buf)
        net.forward(coords, feats)
else:
    s2.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s2):
        net.forward(coords, feats, stream=s2)
    torch.cuda.synchronize()
    spc.spc_set_trace(buf)                 # launch numbering restarts for the captured pass
    with torch.cuda.graph(g, stream=s2):
        net.forward(coords, feats, stream=s2)
    for _ in range(3):
        buf.zero_()
        torch.cuda.synchronize()
        g.replay()
torch.cuda.synchronize()
rec = spc.spc_trace_records(buf)
descs = {L: spc.spc_trace_launch_desc(L) for L in set(rec["launch"].tolist())}
spc.spc_set_trace(None)
if a.out:
    np.save(a.out.replace(".json", "_raw.npy"), rec)
t0 = rec["t"].min()
launches = sorted(set(rec["launch"].tolist()))
rows = []
prev_end = None
print(f"{'launch':>6} {'start':>8} {'gap':>6} {'wait':>6} {'setup':>6} {'rec0':>6} {'full0':>6} {'med':>7} {'end':>7} {'ctas':>5} {'tiles':>5}  desc")
for L in launches:
    r = rec[rec["launch"] == L]
    ev = lambda e: r[r["event"] == e]
    start = ev(0)["t"].min() - t0
    wait = ev(1)["t"].min() - t0
    setup = ev(2)["t"].min() - t0 if len(ev(2)) else wait
    rec0 = ev(3)["t"].min() - t0 if len(ev(3)) else setup
    full0 = ev(4)["t"].min() - t0 if len(ev(4)) else setup
    ends = ev(7)["t"] - t0
    med, end = float(np.median(ends)), float(ends.max())
    tiles = len(ev(6))
    gap = (start - prev_end) if prev_end is not None else 0
    d = descs[L]
    rows.append((L, start, gap, wait, setup, rec0, full0, med, end, len(ends), tiles, d))
    print(f"{L:6d} {start/1e3:8.1f} {gap/1e3:6.1f} {(wait-start)/1e3:6.1f} {(setup-wait)/1e3:6.1f} {(rec0-setup)/1e3:6.1f} "
          f"{(full0-setup)/1e3:6.1f} {(med-start)/1e3:7.1f} {(end-start)/1e3:7.1f} {len(ends):5d} {tiles:5d}  {d}")
    prev_end = end
tot = (rows[-1][8] - rows[0][1]) / 1e3
busy = sum((r[8] - r[1]) for r in rows) / 1e3
print(f"traced span {tot:.1f} us; sum of launch spans {busy:.1f} us; sum of med-exit spans "
      f"{sum((r[7] - r[1]) for r in rows) / 1e3:.1f} us")
if a.out:
    import json
    json.dump({"descs": {int(k): v for k, v in descs.items()}}, open(a.out.replace(".json", "_descs.json"), "w"))
    json.dump([dict(zip(["launch", "start", "gap", "wait", "setup", "rec0", "full0", "med", "end", "ctas", "tiles",
                         "desc"], [int(x) if isinstance(x, (np.integer,)) else (float(x) if not isinstance(x, str) else x)
                                   for x in row])) for row in rows], open(a.out, "w"), indent=0)
