"""A/B timing of one C2 step (captured graph, L2 flushed) for network-level switches.
python scripts/ab_net.py early_maps=0 early_maps=1 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402

coords_np, feats_np, _, _ = bench.workload(0, 2, 1)
n = coords_np.shape[0]
spec = bench.spec_for(coords_np)
dev = torch.device("cuda")
coords = torch.from_numpy(coords_np).to(dev)
feats = torch.zeros(n, C_IN_PAD, dtype=torch.bfloat16, device=dev)
feats[:, :4] = torch.from_numpy(feats_np).to(dev, torch.bfloat16)
flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device=dev)
t_map = bench.load_t(os.path.join(bench.ROOT, "profiles", "r2_tuned_t_c2.json"))
results = {}
for rnd in range(3):
    for arg in sys.argv[1:]:
        k, v = arg.split("=")
        net = SparseNet(n, spec, device=dev)
        net.set_t(t_map)
        if k == "early_maps":
            net.early_maps = bool(int(v))
        elif k == "overlap_proj":
            net.overlap_proj = bool(int(v))
        elif k == "order_max_ts":
            net.order_max_ts = int(v)
            net.density_order = int(v) > 0
        else:
            spc.spc_set_option(getattr(spc, "SPC_OPT_" + k), int(v))
        s2 = torch.cuda.Stream(dev)
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            for _ in range(3):
                net.forward(coords, feats, stream=s2)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s2):
            net.forward(coords, feats, stream=s2)
        ts = []
        for i in range(60):
            flush.fill_(i & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        results.setdefault(arg, []).append(float(np.median(ts[5:])))
        if k not in ("early_maps", "order_max_ts", "overlap_proj"):
            spc.spc_set_option(getattr(spc, "SPC_OPT_" + k), -1)
        del g, net
for k, v in results.items():
    print(f"{k:30s} ms/step {np.round(v, 4).tolist()}  scans/s {1e3 / np.median(v):.1f}")
