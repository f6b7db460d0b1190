"""SURVEY NEXT-3 layer timings on the C2 scan (~99k voxels): K = 2 stride-2 down / up
(offsets {0, s_p}^3) beside the K = 3 layers they replace, a non-cubic (3, 1, 1)
submanifold layer, and spconv's regular K = 3 stride-2 layer (output-site generation +
map + conv) beside the Eq. (1) one.  Per layer: the best dataflow t over all candidates;
CUDA events, median of reps.  JSON lines (profiles/r2_boxes_c2.jsonl).

  python scripts/boxes_bench.py [--c 64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=64)
ap.add_argument("--reps", type=int, default=9)
a = ap.parse_args()

coords = synth.make_scan(2, 0)
spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
fk, _, _ = spc.spc_pack_sort(torch.from_numpy(coords).cuda(), spec)
lv, ln = spc.spc_downsample(fk, spec, [1])
ck = lv[0, :int(ln[0].item())].contiguous()
C = a.c


def med(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def run(name, box, stride, transposed, ik, ok, flags=0, gen=None):
    g = spc.Geom(box, stride, 1, 1, transposed)
    kx, ky, kz = g.box()
    l1max = sum(((k - 1) // 2 if k % 2 else k - 1) for k in (kx, ky, kz))
    F = (torch.rand(ik.shape[0], C, device="cuda") * 2 - 1).bfloat16()
    W = spc.spc_prepare_weight(((torch.rand(g.k_vol(), C, C, device="cuda") * 2 - 1) * 0.05).bfloat16())
    ws = torch.zeros(ok.shape[0] * C * 4 + (1 << 16), dtype=torch.uint8, device="cuda")
    o = torch.empty(ok.shape[0], C, dtype=torch.bfloat16, device="cuda")
    best = None
    for t in range(0, l1max + 2):
        km = spc.spc_build_kmap(ik, ok, spec, g, t, flags)
        nnz = int(spc.spc_kmap_export(km).shape[0])
        us_map = med(lambda: spc.spc_build_kmap(ik, ok, spec, g, t, flags))
        us_conv = med(lambda: spc.spc_conv_forward(km, F, W, C, C, out=o, ws=ws))
        r = {"layer": name, "box": [kx, ky, kz], "stride": stride, "transposed": bool(transposed), "c": C,
             "n_in": int(ik.shape[0]), "n_out": int(ok.shape[0]), "nnz": nnz, "nnz_per_out": round(nnz / ok.shape[0], 3),
             "t": t, "kmap_us": round(us_map, 1), "conv_us": round(us_conv, 1),
             "tflops": round(2.0 * nnz * C * C / (us_conv * 1e-6) / 1e12, 1)}
        if gen is not None:
            r["outputs_us"] = round(gen, 1)
        r["total_us"] = round(us_map + us_conv + (gen or 0.0), 1)
        if best is None or r["total_us"] < best["total_us"]:
            best = r
    print(json.dumps(best), flush=True)


run("down K3 s2 (Eq. 1 sites)", 3, 2, 0, fk, ck)
run("down K2 s2 (TorchSparse)", 2, 2, 0, fk, ck)
run("up K3 s2 transposed", 3, 2, 1, ck, fk)
run("up K2 s2 transposed (TorchSparse)", 2, 2, 1, ck, fk)
run("subm K3", 3, 1, 0, fk, fk, spc.SPC_KMAP_HALVE_SYMMETRIC | spc.SPC_KMAP_DENSITY_ORDER)
run("subm (3,1,1)", (3, 1, 1), 1, 0, fk, fk, spc.SPC_KMAP_HALVE_SYMMETRIC | spc.SPC_KMAP_DENSITY_ORDER)
g = spc.Geom(3, 2, 1, 1, 0)
keys, n_out = spc.spc_regular_outputs(fk, spec, g)
us_gen = med(lambda: spc.spc_regular_outputs(fk, spec, g))
rk = keys[:int(n_out.item())].contiguous()
run("down K3 s2 (spconv regular sites)", 3, 2, 0, fk, rk, gen=us_gen)
