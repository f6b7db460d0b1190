"""NEXT-1 ablation ("negligible performance impact" of 64- vs 32-bit packing): the
C2 scan (bits 0/12/11/8 = 31, fits 32) packed + sorted and its level-0 submanifold,
strided and transposed K=3 maps built with 64-bit and with 32-bit keys (identical maps,
checked), timed with CUDA events (median, L2 flushed).  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

coords_np, _, _, _ = bench.workload(0, 2, 1)
spec = bench.spec_for(coords_np)
assert spec.used_bits() <= 32
dev = torch.device("cuda")
coords = torch.from_numpy(coords_np).to(dev)
flush = torch.empty(320 * 2 ** 20, dtype=torch.uint8, device=dev)
ALL = spc.SPC_KMAP_HALVE_SYMMETRIC | spc.SPC_KMAP_DENSITY_ORDER


def med(fn, reps=30):
    fn()
    torch.cuda.synchronize()
    out = []
    for r in range(reps):
        flush.fill_(r & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return float(np.median(out))


res = {}
maps = {}
for bits in (64, 32):
    n = coords.shape[0]
    kt = torch.int32 if bits == 32 else torch.int64
    keys = torch.empty(n, dtype=kt, device=dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    ws = torch.empty(int(spc.lib().spc_pack_sort_workspace_size(n)), dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    res[f"pack_sort_us_{bits}"] = med(lambda: spc.spc_pack_sort(coords, spec, status=st, keys_out=keys, perm_out=perm,
                                                                ws=ws, key_bits=bits))
    lv, ln = spc.spc_downsample(spc.spc_pack_sort(coords, spec)[0], spec, [1])
    coarse64 = lv[0, :int(ln[0].item())].contiguous()
    coarse = coarse64.to(torch.int32) if bits == 32 else coarse64   # (keys < 2^31: exact)
    for name, (ik, ok, g, t, fl) in {"subm": (keys, keys, spc.Geom(3, 1, 1, 1, 0), 4, ALL),
                                     "strided": (keys, coarse, spc.Geom(3, 2, 1, 1, 0), 4, spc.SPC_KMAP_DENSITY_ORDER),
                                     "transposed": (coarse, keys, spc.Geom(3, 2, 1, 1, 1), 4,
                                                    spc.SPC_KMAP_DENSITY_ORDER)}.items():
        buf = torch.empty(spc.spc_kmap_bytes(g, t, fl, ik.shape[0], ok.shape[0]) + 256, dtype=torch.uint8, device=dev)
        res[f"kmap_{name}_us_{bits}"] = med(lambda: spc.spc_build_kmap(ik, ok, spec, g, t, fl, buf=buf))
        maps[(name, bits)] = spc.spc_kmap_export(spc.spc_build_kmap(ik, ok, spec, g, t, fl))
for name in ("subm", "strided", "transposed"):
    assert np.array_equal(maps[(name, 64)], maps[(name, 32)]), name
res["index_total_us_64"] = sum(v for k, v in res.items() if k.endswith("_64"))
res["index_total_us_32"] = sum(v for k, v in res.items() if k.endswith("_32") and not k.startswith("index"))
print(json.dumps({"what": "NEXT-1: 64- vs 32-bit packed keys on the C2 scan (P:518)", "n_voxels": int(coords.shape[0]),
                  "pack_spec": list(spec.astuple()), "maps_identical": True,
                  **{k: round(v, 1) for k, v in res.items()},
                  "speedup_32_over_64": round(res["index_total_us_64"] / res["index_total_us_32"], 3),
                  "paper": "negligible performance impact of 64-bit packing (P:518); 1.3% vs 1.6% pack+sort share (P:519)"}))
