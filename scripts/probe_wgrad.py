"""Probe of the training kernels on one C2-level map: spc_conv_wgrad (on the all-WS halved
map the network's backward uses, and on the all-OS forward map) and the dgrad convolution,
CUDA events over repeated launches.  python scripts/probe_wgrad.py [--level L] [--cin C] [--cout C]"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--cin", type=int, default=32)
    ap.add_argument("--cout", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ipsm", type=int, default=-1)
    args = ap.parse_args()
    spc.spc_set_option(spc.SPC_OPT_WGRAD_ITEMS_PER_SM, args.ipsm)
    coords, _, _, _ = bench.workload(0, 2)
    spec = bench.spec_for(coords)
    keys, _, _ = spc.spc_pack_sort(torch.from_numpy(coords).cuda(), spec)
    if args.level > 0:
        lv, ln = spc.spc_downsample(keys, spec, [args.level])
        keys = lv[0, :int(ln[0].item())].contiguous()
    n = keys.shape[0]
    g = spc.Geom(3, 1, 1, 2 ** args.level, 0)
    km_ws = spc.spc_build_kmap(keys, keys, spec, g, 0, spc.SPC_KMAP_HALVE_SYMMETRIC)
    km_os = spc.spc_build_kmap(keys, keys, spec, g, -1, spc.SPC_KMAP_HALVE_SYMMETRIC | spc.SPC_KMAP_DENSITY_ORDER)
    F = torch.from_numpy(synth.make_features(n, args.cin, seed=1)).cuda().bfloat16()
    G = torch.from_numpy(synth.make_features(n, args.cout, seed=2)).cuda().bfloat16()
    W = torch.from_numpy(synth.make_weights(27, args.cin, args.cout, seed=3, nnz_per_out=6)).cuda().bfloat16()
    Wf = spc.spc_prepare_weight(W)
    Wd = spc.spc_prepare_weight_ex(W, spc.SPC_WEIGHT_DGRAD_MIRROR)
    dW = torch.zeros(27, args.cin, args.cout, dtype=torch.float32, device="cuda")
    out = torch.empty(n, args.cout, dtype=torch.bfloat16, device="cuda")
    dF = torch.empty(n, args.cin, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(spc.spc_conv_workspace_size(km_os, max(args.cin, args.cout)) + 2 ** 20, dtype=torch.uint8,
                     device="cuda")
    nnz = int(spc.spc_kmap_export(km_os).shape[0])
    fl = 2.0 * nnz * args.cin * args.cout
    r = {}
    r["fwd_os"] = timed(lambda: spc.spc_conv_forward(km_os, F, Wf, args.cin, args.cout, out=out, ws=ws), args.reps)
    r["dgrad_os"] = timed(lambda: spc.spc_conv_forward(km_os, G, Wd, args.cout, args.cin, out=dF, ws=ws), args.reps)
    r["wgrad_ws"] = timed(lambda: spc.spc_conv_wgrad(km_ws, F, G, args.cin, args.cout, d_weight=dW), args.reps)
    r["wgrad_os"] = timed(lambda: spc.spc_conv_wgrad(km_os, F, G, args.cin, args.cout, d_weight=dW), args.reps)
    print(f"ipsm={args.ipsm} level={args.level} n={n} nnz={nnz} cin={args.cin} cout={args.cout} " +
          " ".join(f"{k}={v:.1f}us({fl / v / 1e6:.0f}TF/s)" for k, v in r.items()), flush=True)


if __name__ == "__main__":
    main()
