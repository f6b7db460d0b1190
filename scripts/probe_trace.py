"""Per-stage device trace of one wide layer (spc_set_trace fine events, CTAs 0 and 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

cin, cout, t, pair = (int(v) for v in sys.argv[1:5])
out_npy = sys.argv[5]
spc.spc_set_option(spc.SPC_OPT_CONV_CTA_PAIR, pair)
coords = synth.make_scan(5, 0)
spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
keys, perm, _ = spc.spc_pack_sort(torch.from_numpy(coords).cuda(), spec)
km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), t, spc.SPC_KMAP_HALVE_SYMMETRIC | spc.SPC_KMAP_DENSITY_ORDER)
n = keys.shape[0]
F = torch.randn(n, cin, device="cuda").bfloat16()
W = spc.spc_prepare_weight((torch.randn(27, cin, cout, device="cuda") * 0.05).bfloat16())
out = torch.empty(n, cout, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(spc.spc_conv_workspace_size(km, cout), dtype=torch.uint8, device="cuda")
for _ in range(3):
    spc.spc_conv_forward(km, F, W, cin, cout, out=out, ws=ws)
buf = torch.zeros(1 + 2 * 2_000_000, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
spc.spc_set_trace(buf)
spc.spc_conv_forward(km, F, W, cin, cout, out=out, ws=ws)
torch.cuda.synchronize()
rec = spc.spc_trace_records(buf)
spc.spc_set_trace(None)
np.save(out_npy, rec)
print("records", len(rec))
