"""Two scans in flight (serving pipeline probe): step i runs the feature computation of
scan i on at most `cap` SMs (SPC_OPT_CONV_MAX_CTAS) while the voxel indexing of scan i+1
runs on another stream; two SparseNet instances alternate.  Captured as two CUDA graphs
(one per parity), L2 flushed before every step, CUDA events; compared with the sequential
forward.  python scripts/pipeline_probe.py [--config 2] [--caps 0 136 128 120]"""
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


def timed(replays, flush, n=40):
    ts = []
    for i in range(n):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        replays[i % len(replays)].replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[4:]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--caps", type=int, nargs="+", default=[0])
    ap.add_argument("--prios", type=int, nargs="+", default=[0],
                    help="conv-stream priorities (< 0 = higher); the indexing stream stays at 0")
    ap.add_argument("--afters", type=int, nargs="+", default=[19])
    ap.add_argument("--index-afters", type=int, nargs="+", default=[-1])
    ap.add_argument("--t-set", action="append", default=[],
                    help="K,stride,ts,tr=t overrides on top of the tuned t (e.g. 3,1,8,0=4)")
    ap.add_argument("--caps3", nargs="+", default=["0"],
                    help="SPC_OPT_CONV_MAX_CTAS while capturing the three- / four-deep pipelines "
                         "(one value, or comma-separated per segment)")
    ap.add_argument("--t-from", default=None, help="tuned t file (bench.py --save-t); default: C2's committed one")
    ap.add_argument("--splitsets", nargs="+", default=["22", "15,30", "13,26", "19,34", "10,25", "22,36"],
                    help="comma-separated split layers (one: three scans in flight, two: four)")
    args = ap.parse_args()
    dev = torch.device("cuda")
    coords_np, feats_np, _, net_name = bench.workload(0, args.config)
    spec = bench.spec_for(coords_np)
    t_map = bench.load_t(args.t_from) if args.t_from else \
        (bench.load_t(os.path.join(ROOT, "profiles", "r2_tuned_t_c2.json")) if args.config == 2 else None)
    for o in args.t_set:
        k, v = o.split("=")
        t_map = dict(t_map or {})
        t_map[tuple(int(x) for x in k.split(","))] = int(v)
    nets = []
    for _ in range(2):
        net = SparseNet(coords_np.shape[0], spec, net=net_name)
        if t_map:
            net.set_t(t_map)
        nets.append(net)
    coords = torch.from_numpy(coords_np).to(dev)
    feats = torch.zeros(coords_np.shape[0], C_IN_PAD, dtype=torch.bfloat16, device=dev)
    feats[:, :feats_np.shape[1]] = torch.from_numpy(feats_np).to(dev).bfloat16()
    for net in nets:
        for _ in range(2):
            net.forward(coords, feats)
    torch.cuda.synchronize()
    flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device=dev)
    s0, s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    # sequential reference: one graph of the whole forward
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s0):
        nets[0].forward(coords, feats, stream=s0)
    torch.cuda.synchronize()
    res = {"sequential_ms": timed([g], flush)}
    ref = nets[0].bufs[nets[0].out_name].float().clone()
    g.replay()
    torch.cuda.synchronize()
    # fp32 atomics in the weight-stationary layers: runs agree to rounding, not bit-for-bit
    res["sequential_run_to_run_maxdiff"] = float((nets[0].bufs[nets[0].out_name].float() - ref).abs().max())
    from paper_2511_20834_b200.network import capture_pipeline  # noqa: F811
    for cap in args.caps:
        for prio in args.prios:
            for after in args.afters:
                spc.spc_set_option(spc.SPC_OPT_CONV_MAX_CTAS, cap)
                graphs = capture_pipeline(nets, [(coords, feats), (coords, feats)], dev, torch.cuda.current_stream(),
                                          conv_priority=prio, index_after_layer=after)
                spc.spc_set_option(spc.SPC_OPT_CONV_MAX_CTAS, -1)
                key = f"cap{cap}_prio{prio}_after{after}"
                res["ms_" + key] = timed(graphs, flush)
                res["maxdiff_" + key] = max(float((nets[q].bufs[nets[q].out_name].float() - ref).abs().max())
                                            for q in range(2))
    # three and four scans in flight
    from paper_2511_20834_b200.network import capture_pipeline_n
    extra = []
    for _ in range(2):
        nt = SparseNet(coords_np.shape[0], spec, net=net_name)
        if t_map:
            nt.set_t(t_map)
        for _ in range(2):
            nt.forward(coords, feats)
        extra.append(nt)
    torch.cuda.synchronize()
    for sp in args.splitsets:
        splits = [int(v) for v in sp.split(",")]
        D = len(splits) + 2
        nn = (nets + extra)[:D]
        for ia in args.index_afters:
            for cap in args.caps3:
                cv = [int(x) for x in cap.split(",")]
                graphs = capture_pipeline_n(nn, [(coords, feats)] * D, dev, torch.cuda.current_stream(), splits,
                                            index_after_layer=ia, conv_max_ctas=cv if len(cv) > 1 else cv[0])
                res[f"ms_split{sp}_ia{ia}_cap{cap}"] = timed(graphs, flush, n=60)
    print(json.dumps({"config": args.config, "n": int(coords_np.shape[0]), **res}))


if __name__ == "__main__":
    main()
