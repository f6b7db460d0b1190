"""First-tile event timeline of one k_conv_tc launch (SPC_EXP_TRACE3 build):
python -m paper_2511_20834_b200.build --exp TF -DSPC_EXP_TRACE3
SPC_LIB_OVERRIDE=paper_2511_20834_b200/exp_TF.so python scripts/timeline_first.py --cin 64 --cout 64 --t -1 --n 20000
"""
import ctypes, os, sys, runpy
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("SPC_LIB_OVERRIDE", os.path.join(here, "..", "paper_2511_20834_b200", "exp_TF.so"))
sys.argv = ["probe_conv.py"] + sys.argv[1:] + ["--reps", "1"]
import paper_2511_20834_b200 as spc
L = spc.lib()
L.spc_exp_tl_read.argtypes = [ctypes.c_void_p]
g = runpy.run_path(os.path.join(here, "probe_conv.py"), run_name="__main__")
import torch
torch.cuda.synchronize()
L.spc_exp_tl_clear()
g["spc"].spc_conv_forward(g["km"], g["F"], g["W"], g["a"].cin, g["a"].cout, out=g["out"], ws=g["ws"])
torch.cuda.synchronize()
buf = np.zeros((8, 1024), np.uint64)
L.spc_exp_tl_read(buf.ctypes.data)
n = int((buf[0] > 0).sum())
t = buf[:, :n].astype(np.int64)
t0 = t[0].min()
names = ["entry", "setup", "sched_decoded", "sched_record", "gather_blk", "gather_issued", "weights_issued", "mma_full"]
for i, nm in enumerate(names):
    v = t[i][t[i] > 0]
    if len(v):
        r = (v - t0) / 1000.0
        print(f"  {nm:15s} min {r.min():7.2f}  median {np.median(r):7.2f}  max {r.max():7.2f}  (n={len(v)})")
