"""One forward pass of a bench network inside a cudaProfilerStart/Stop region (for ncu with
--profile-from-start off): the same workload, weights and per-map dataflow t as bench.py.

python scripts/one_pass.py [--config 2|3|4] [--t-from gpurun_out/bench.json]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD  # noqa: E402
import paper_2511_20834_b200 as spc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--t-from", default=None)
a = ap.parse_args()

coords_np, feats_np, _, net_name = bench.workload(0, a.config, 1)
n = coords_np.shape[0]
spec = bench.spec_for(coords_np) if a.config != 4 else spc.spc_plan_pack(
    coords_np[:, 1:].min(0), coords_np[:, 1:].max(0), 8, 16, 16)
net = SparseNet(n, spec, net=net_name)
if a.t_from:
    net.set_t(bench.load_t(a.t_from))
coords = torch.from_numpy(coords_np).cuda()
feats = torch.zeros(n, C_IN_PAD, dtype=torch.bfloat16, device="cuda")
feats[:, :feats_np.shape[1]] = torch.from_numpy(feats_np).cuda().bfloat16()
for _ in range(3):
    net.forward(coords, feats)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
net.forward(coords, feats)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("layers:", [(s.name, s.map_key, s.c_in, s.c_out) for s in net.layers])
