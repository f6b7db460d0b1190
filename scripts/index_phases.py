"""In-graph timing of the indexing phase's parts on one scan (CUDA graphs, CUDA events,
L2 flushed between replays): pack+sort, row gather, downsample (all levels), and the
network-wide map build (spc_network_kmaps = downsample + every map + density order).

python scripts/index_phases.py [--config 2]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402


def graph_time(fn, reps=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    torch.cuda.synchronize()
    flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    coords_np, feats_np, _, net_name = bench.workload(0, args.config)
    spec = bench.spec_for(coords_np)
    net = SparseNet(coords_np.shape[0], spec, net=net_name)
    bench_t = os.path.join(ROOT, "profiles", "r2_tuned_t_c2.json")
    if args.config == 2 and os.path.exists(bench_t):
        net.set_t(bench.load_t(bench_t))
    c = torch.from_numpy(coords_np).cuda()
    f = torch.zeros(coords_np.shape[0], C_IN_PAD, dtype=torch.bfloat16, device="cuda")
    n = c.shape[0]
    net.forward(c, f)   # allocate everything once
    torch.cuda.synchronize()
    r = {}
    r["pack_sort"] = graph_time(lambda s: spc.spc_pack_sort(c, spec, status=net.status, keys_out=net.keys[:n],
                                                             perm_out=net.perm[:n], ws=net.sort_ws, stream=s))
    r["gather_rows"] = graph_time(lambda s: spc.spc_gather_rows(f, net.perm[:n], out=net.bufs["x0"][:n], stream=s))
    levels = list(range(1, net.n_levels))
    ds_out = torch.empty((len(levels), n), dtype=torch.int64, device="cuda")
    ds_n = torch.empty(len(levels), dtype=torch.int64, device="cuda")
    ds_ws = torch.empty(int(spc.lib().spc_downsample_workspace_size(n, len(levels))), dtype=torch.uint8, device="cuda")
    L = (spc.ctypes.c_int32 * len(levels))(*levels)

    def ds(s):
        spc._check(spc.lib().spc_downsample(spc._ptr(net.keys), n, None, spec, len(levels), L, spc._ptr(ds_out),
                                            spc._ptr(ds_n), spc._ptr(ds_ws), ds_ws.numel(), spc._stream(s)),
                   "spc_downsample")
    r["downsample"] = graph_time(ds)
    r["network_kmaps"] = graph_time(lambda s: net.index(stream=s))
    r["maps_only_est"] = r["network_kmaps"] - r["downsample"]
    print(json.dumps({"config": args.config, "n": n, "maps": len(net.map_keys), "us": r}))


if __name__ == "__main__":
    main()
