"""Time the voxel-indexing calls of one C2 scan (pack+sort, downsample, each kernel map)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2511_20834_b200 as spc

coords = synth.make_scan(int(os.environ.get("CFG", 2)), 0)
n = coords.shape[0]
spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
c = torch.from_numpy(coords).cuda()


def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


keys = torch.empty(n, dtype=torch.int64, device="cuda"); perm = torch.empty(n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(spc.lib().spc_pack_sort_workspace_size(n)), dtype=torch.uint8, device="cuda")
print(f"n={n} pack_sort: {timeit(lambda: spc.spc_pack_sort(c, spec, keys_out=keys, perm_out=perm, ws=ws)):.1f} us")
print(f"downsample x4: {timeit(lambda: spc.spc_downsample(keys, spec, [1, 2, 3, 4])):.1f} us")
lv, ln = spc.spc_downsample(keys, spec, [1, 2, 3, 4])
ln = ln.cpu().tolist()
levels = [keys] + [lv[i, :ln[i]] for i in range(4)]
for (K, s, l, t, fl, tr) in [(3, 1, 0, -1, 0, 0), (3, 1, 0, 0, 1, 0), (3, 1, 0, 2, 1, 0), (3, 2, 0, -1, 0, 0),
                              (3, 2, 0, -1, 0, 1), (3, 1, 1, -1, 0, 0), (3, 1, 2, -1, 0, 0), (5, 1, 0, 3, 1, 0)]:
    if tr:
        inp, out = levels[l + 1], levels[l]
    elif s == 2:
        inp, out = levels[l], levels[l + 1]
    else:
        inp = out = levels[l]
    g = spc.Geom(K, s, 1, 2 ** l, tr)
    km = spc.spc_build_kmap(inp, out, spec, g, t, fl)
    us = timeit(lambda: spc.spc_build_kmap(inp, out, spec, g, t, fl))
    print(f"kmap K={K} s={s} lvl={l} t={t} halve={fl} tr={tr} n_out={out.shape[0]}: {us:.1f} us")
from paper_2511_20834_b200.network import SparseUNet
net = SparseUNet(n, spec)
net.keys.copy_(keys)
net.index()
print(f"network_kmaps (MinkUNet, {len(net.map_keys)} maps): {timeit(lambda: net.index()):.1f} us")
