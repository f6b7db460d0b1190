"""compute-sanitizer target: the whole hot path on the C1 scan -- pack+sort,
gather, network-wide indexing (5 levels, 18 maps, density order), the 49 MinkUNet-42
convolutions (OS, WS, hybrid, split-K) -- plus standalone map builds and conv calls that
exercise the WS / split / 256-row / fp32 paths.

  compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_c1.py [--small]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402

small = "--small" in sys.argv
coords = synth.make_scan(1, 0)
if small:
    coords = coords[:3000]
n = coords.shape[0]
spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
dev = torch.device("cuda")
c = torch.from_numpy(coords).to(dev)
feats = torch.zeros(n, C_IN_PAD, dtype=torch.bfloat16, device=dev)
feats[:, :4] = torch.from_numpy(synth.make_features(n, 4, seed=1)).to(dev).bfloat16()
for t_map in (None, {(3, 1, 1, 0): 0, (3, 1, 2, 0): -1, (3, 2, 1, 0): 2}):
    net = SparseNet(n, spec, device=dev, t_override=t_map)
    net.forward(c, feats)
    torch.cuda.synchronize()
    assert int(net.status.item()) == 0
keys, perm, _ = spc.spc_pack_sort(c, spec)
for t, fl, ci, co, dt in ((-1, 0, 64, 256, torch.bfloat16), (2, 9, 32, 64, torch.bfloat16), (0, 1, 16, 32, torch.float32),
                          (3, 9, 32, 32, torch.bfloat16)):
    K = 5 if t == 3 else 3
    km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(K, 1, 1, 1, 0), t, fl)
    F = torch.randn(n, ci, device=dev).to(dt)
    W = spc.spc_prepare_weight((torch.randn(K ** 3, ci, co, device=dev) * 0.05).to(dt))
    out = spc.spc_conv_forward(km, F, W, ci, co, out_dtype=torch.float32 if dt == torch.float32 else torch.bfloat16)
torch.cuda.synchronize()
# one training step (dgrad through the forward kernels, wgrad, residual adds)
# and the fused BN / ReLU epilogue
tnet = SparseNet(n, spec, device=dev, train=True)
tnet.forward(c, feats)
tnet.backward(torch.randn(n, tnet.bufs[tnet.out_name].shape[1], device=dev).bfloat16())
km = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), 2, 9)
F = torch.randn(n, 64, device=dev).bfloat16()
W = spc.spc_prepare_weight((torch.randn(27, 64, 96, device=dev) * 0.05).bfloat16())
sc, sh = torch.rand(96, device=dev) + 0.5, torch.randn(96, device=dev)
spc.spc_conv_forward(km, F, W, 64, 96, out_dtype=torch.bfloat16, residual=torch.randn(n, 96, device=dev).bfloat16(),
                     scale=sc, shift=sh, relu=True)
for tt in (-1, 0):
    kw = spc.spc_build_kmap(keys, keys, spec, spc.Geom(3, 1, 1, 1, 0), tt, 1)
    spc.spc_conv_wgrad(kw, F, torch.randn(n, 96, device=dev).bfloat16(), 64, 96)
    spc.spc_conv_wgrad(kw, F.float()[:, :32].contiguous(), torch.randn(n, 16, device=dev), 32, 16)
torch.cuda.synchronize()
print("sanitize target done", n)
