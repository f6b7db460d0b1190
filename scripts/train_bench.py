"""SURVEY NEXT-4 measurement: one MinkUNet-42 training step on the C2 scan (forward +
backward: every layer's wgrad, dgrad and residual branch) through libspc, captured as one
CUDA graph, L2 flushed (320 MB write) between timed steps, CUDA events.  Also an
instrumented pass with events around each layer's backward calls (us and algorithmic
TFLOP/s: dgrad and wgrad each 2 * nnz * C_in * C_out, like the forward).

python scripts/train_bench.py [--config 2] [--steps 20] [--warmup 5] [--t-from profiles/r2_tuned_t_c2.json]
prints one JSON line (kept under profiles/)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (workload / spec_for / Clocks: same synthetic inputs as the bench)
import paper_2511_20834_b200 as spc  # noqa: E402
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--t-from", default=os.path.join(ROOT, "profiles", "r2_tuned_t_c2.json"))
    ap.add_argument("--opt", action="append", default=[], help="NAME=VALUE spc_set_option (A/B runs)")
    args = ap.parse_args()
    for o in args.opt:
        k, v = o.split("=")
        spc.spc_set_option(getattr(spc, "SPC_OPT_" + k), int(v))
    dev = torch.device("cuda:0")
    coords_np, feats_np, _, net_name = bench.workload(0, args.config)
    spec = bench.spec_for(coords_np)
    net = SparseNet(coords_np.shape[0], spec, net=net_name, train=True)
    if args.t_from and os.path.exists(args.t_from):
        # the forward maps take the bench's tuned t; the extra dgrad maps keep their default
        net.set_t({mk: t for mk, t in bench.load_t(args.t_from).items() if mk in net.t})
    coords = torch.from_numpy(coords_np).to(dev)
    feats = torch.zeros(coords_np.shape[0], C_IN_PAD, dtype=torch.bfloat16, device=dev)
    feats[:, :feats_np.shape[1]] = torch.from_numpy(feats_np).to(dev).bfloat16()
    gout = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (coords_np.shape[0], net.bufs[net.out_name].shape[1]))
                            .astype(np.float32)).to(dev).bfloat16()
    stream = torch.cuda.current_stream(dev)

    def fwd(st):
        net.forward(coords, feats, stream=st)

    def bwd(st):
        net.backward(gout, stream=st)

    for _ in range(3):
        fwd(stream)
        bwd(stream)
    torch.cuda.synchronize()
    s2 = torch.cuda.Stream(dev)
    s2.wait_stream(stream)
    graphs = {}
    for name, fn in (("fwd", fwd), ("bwd", bwd)):
        with torch.cuda.stream(s2):
            fn(s2)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s2):
            fn(s2)
        torch.cuda.synchronize()
        graphs[name] = g
    flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        graphs["fwd"].replay()
        graphs["bwd"].replay()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    with bench.Clocks(0) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            graphs["fwd"].replay()
            ev[i][1].record(stream)
            graphs["bwd"].replay()
            ev[i][2].record(stream)
        torch.cuda.synchronize()
    f_ms = float(np.median([a.elapsed_time(b) for a, b, _ in ev]))
    b_ms = float(np.median([b.elapsed_time(c) for _, b, c in ev]))
    # two scans in flight: the next scan's voxel indexing (second training instance, its own
    # stream) beside this scan's convolutions + backward
    net2 = SparseNet(coords_np.shape[0], spec, net=net_name, train=True)
    net2.set_t(dict(net.t))
    for _ in range(2):
        net2.forward(coords, feats)
        net2.backward(gout)
    torch.cuda.synchronize()
    nets = [net, net2]
    sA, sB, sC = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    pg = []
    for p in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=sA):
            fork = torch.cuda.Event()
            fork.record(sA)
            sB.wait_event(fork)
            sC.wait_event(fork)
            with torch.cuda.stream(sB):
                nets[p].conv_stage(sB)
                nets[p].backward(gout, stream=sB)
            with torch.cuda.stream(sC):
                nets[1 - p].index_stage(coords, feats, sC)
            j1, j2 = torch.cuda.Event(), torch.cuda.Event()
            j1.record(sB)
            j2.record(sC)
            sA.wait_event(j1)
            sA.wait_event(j2)
        torch.cuda.synchronize()
        pg.append(g)
    pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        pev[i][0].record(stream)
        pg[i % 2].replay()
        pev[i][1].record(stream)
    torch.cuda.synchronize()
    p_ms = float(np.median([a.elapsed_time(b) for a, b in pev]))
    # instrumented pass: per-layer backward (wgrad + residual + dgrad) with events
    flops = net.algorithmic_flops()
    net.backward(gout)   # zero / seed the gradient buffers
    torch.cuda.synchronize()
    layers = []
    for i in reversed(range(len(net.layers))):
        s = net.layers[i]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        net.backward_layer(i)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3
        fl = flops[s.name] * (2 if i > 0 else 1)   # wgrad (+ dgrad)
        layers.append({"name": s.name, "c_in": s.c_in, "c_out": s.c_out, "us": round(us, 2),
                       "gflop": round(fl / 1e9, 4), "tflops": round(fl / us / 1e6, 2)})
    fwd_fl = sum(flops.values())
    bwd_fl = sum(flops[s.name] * (2 if i > 0 else 1) for i, s in enumerate(net.layers))
    line = {"metric": "MinkUNet training steps/s (forward + backward, per scan)", "value": 1e3 / p_ms,
            "pipeline": "two scans in flight: the next scan's voxel indexing beside this scan's convolutions "
                        "and backward (second training instance, own stream)",
            "sequential": {"value": 1e3 / (f_ms + b_ms), "ms_per_step": f_ms + b_ms},
            "unit": "steps/s", "config": {"workload": f"C{args.config} {net_name}, one synthetic scan, random bf16 "
                                                      "weights, random bf16 output gradient", "n_voxels": int(coords_np.shape[0]),
                                          "l2": "flushed (320 MB write) between timed steps", "cuda_graph": True},
            "forward_ms": f_ms, "backward_ms": b_ms, "forward_tflops": fwd_fl / f_ms / 1e9,
            "backward_tflops": bwd_fl / b_ms / 1e9, "backward_gflop": bwd_fl / 1e9, "dtype": "bf16",
            "clocks": clk.summary(), "layers": layers[::-1]}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
