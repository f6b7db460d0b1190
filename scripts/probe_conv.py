"""Run one sparse-conv layer of config C2 repeatedly (for ncu / timing probes).

python scripts/probe_conv.py --cin 96 --cout 96 --t -1 --level 0 --reps 5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cin", type=int, default=96)
ap.add_argument("--cout", type=int, default=96)
ap.add_argument("--K", type=int, default=3)
ap.add_argument("--t", type=int, default=-1)
ap.add_argument("--halve", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=0, help="keep the first n points of the scan")
ap.add_argument("--order", type=int, default=1, help="SPC_KMAP_DENSITY_ORDER")
ap.add_argument("--pair", type=int, default=-1, help="SPC_OPT_CONV_CTA_PAIR (0 off, 1 auto, 2 force; -1 default)")
ap.add_argument("--opt", action="append", default=[], help="NAME=VALUE spc_set_option (e.g. CONV_STAGE_KB=96)")
a = ap.parse_args()
spc.spc_set_option(spc.SPC_OPT_CONV_CTA_PAIR, a.pair)
for o in a.opt:
    k, v = o.split("=")
    spc.spc_set_option(getattr(spc, "SPC_OPT_" + k), int(v))

coords = synth.make_scan(a.config, 0)
if a.n:
    coords = coords[:a.n]
spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
keys, perm, _ = spc.spc_pack_sort(torch.from_numpy(coords).cuda(), spec)
km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(a.K, 1, 1, 1, 0), a.t,
                        (spc.SPC_KMAP_HALVE_SYMMETRIC if a.halve else 0) | (spc.SPC_KMAP_DENSITY_ORDER if a.order else 0))
n = keys.shape[0]
F = torch.randn(n, a.cin, device="cuda").bfloat16()
W = spc.spc_prepare_weight((torch.randn(a.K ** 3, a.cin, a.cout, device="cuda") * 0.05).bfloat16())
out = torch.empty(n, a.cout, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(spc.spc_conv_workspace_size(km, a.cout), dtype=torch.uint8, device="cuda")
nnz = spc.spc_kmap_export(km).shape[0]
for _ in range(2):
    spc.spc_conv_forward(km, F, W, a.cin, a.cout, out=out, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    spc.spc_conv_forward(km, F, W, a.cin, a.cout, out=out, ws=ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
fl = 2.0 * nnz * a.cin * a.cout
print(f"n={n} nnz={nnz} k_dense={km.k_dense} lists={km.n_lists} cin={a.cin} cout={a.cout} t={a.t} pair={a.pair}: "
      f"{ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s (algorithmic)")
if os.environ.get("PROBE_KERNELS"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            spc.spc_conv_forward(km, F, W, a.cin, a.cout, out=out, ws=ws)
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if "CUDA" in str(getattr(e, "device_type", ""))], key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    for e in ev:
        print(f"  {e.name.split('(')[0][:40]:40s} start {e.time_range.start - t0:8.1f} dur {e.time_range.elapsed_us():7.1f}")
