"""C5 layer-wise sweep: one KITTI-shaped ~100k-voxel scan; channels 16-256,
K 3/5, layer stride 1/2, every dataflow threshold t (0 = all WS ... L1max+1 = all OS).
Times kernel-map build + feature computation with CUDA events (median of reps), prints
JSON lines and writes a markdown table (argv[1], default profiles/c5_sweep.md)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

out_md = sys.argv[1] if len(sys.argv) > 1 else "profiles/c5_sweep.md"
coords = synth.make_scan(5, 0)
spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
keys, perm, _ = spc.spc_pack_sort(torch.from_numpy(coords).cuda(), spec)
lv, ln = spc.spc_downsample(keys, spec, [1])
n1 = int(ln[0].item())
coarse = lv[0, :n1].contiguous()
ws = torch.zeros(keys.shape[0] * 256 * 4 + (1 << 16), dtype=torch.uint8, device="cuda")   # accumulator + tile counters


def med(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


rows = []
for (ci, co) in [(16, 16), (16, 32), (32, 32), (64, 64), (128, 128), (256, 256)]:
    for K in (3, 5):
        for sl in (1, 2):
            inp, out = keys, (keys if sl == 1 else coarse)
            g = spc.Geom(K, sl, 1, 1, 0)
            F = (torch.rand(inp.shape[0], ci, device="cuda") * 2 - 1).bfloat16()
            W = spc.spc_prepare_weight(((torch.rand(K ** 3, ci, co, device="cuda") * 2 - 1) * 0.05).bfloat16())
            o = torch.empty(out.shape[0], co, dtype=torch.bfloat16, device="cuda")
            l1max = 3 * (K - 1) // 2
            best = None
            for t, ordered in [(t, o) for t in range(0, l1max + 2) for o in ((False, True) if t > 0 else (False,))]:
                fl = spc.SPC_KMAP_HALVE_SYMMETRIC if sl == 1 else 0
                if ordered:   # the density order of the OS part (what the network bench builds)
                    fl |= spc.SPC_KMAP_DENSITY_ORDER
                km = spc.spc_build_kmap(inp, out, spec, g, t, fl)
                nnz = int(km.counts()[:K ** 3].sum().item())
                if sl == 1 and fl:   # halved maps do not count mirror offsets beyond the centre
                    nnz = int(spc.spc_kmap_export(km).shape[0])
                us_map = med(lambda: spc.spc_build_kmap(inp, out, spec, g, t, fl))
                us_conv = med(lambda: spc.spc_conv_forward(km, F, W, ci, co, out=o, ws=ws))
                fl_ = 2.0 * nnz * ci * co
                kind = ("WS" if t == 0 else ("OS" if t == l1max + 1 else f"hybrid t={t}")) + (" +ord" if ordered else "")
                r = {"c_in": ci, "c_out": co, "K": K, "stride": sl, "t": t, "dataflow": kind, "nnz": nnz,
                     "kmap_us": round(us_map, 1), "conv_us": round(us_conv, 1), "total_us": round(us_map + us_conv, 1),
                     "tflops": round(fl_ / (us_conv * 1e-6) / 1e12, 1), "k_dense": km.k_dense, "n_lists": km.n_lists}
                print(json.dumps(r), flush=True)
                rows.append(r)
os.makedirs(os.path.dirname(out_md) or ".", exist_ok=True)
with open(out_md, "w") as f:
    f.write("# C5 layer sweep (B200, one KITTI-shaped scan, %d voxels; stride-2 outputs: %d)\n\n" % (keys.shape[0], n1))
    f.write("kmap = spc_build_kmap; conv = spc_conv_forward (bf16 in/out, fp32 accumulate); TFLOP/s = 2 nnz Cin Cout / conv time; +ord = SPC_KMAP_DENSITY_ORDER (the OS part in density order, as the network builds it; its kmap time includes the order).\n\n")
    f.write("| C_in | C_out | K | s | dataflow | kmap us | conv us | total us | TFLOP/s | best |\n|---|---|---|---|---|---|---|---|---|---|\n")
    groups = {}
    for r in rows:
        groups.setdefault((r["c_in"], r["c_out"], r["K"], r["stride"]), []).append(r)
    for key, rs in groups.items():
        bt = min(rs, key=lambda r: r["total_us"])
        for r in rs:
            f.write(f"| {r['c_in']} | {r['c_out']} | {r['K']} | {r['stride']} | {r['dataflow']} | {r['kmap_us']} | "
                    f"{r['conv_us']} | {r['total_us']} | {r['tflops']} | {'**best**' if r is bt else ''} |\n")
print("wrote", out_md)
