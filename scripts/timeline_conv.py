"""Per-CTA timeline of one k_conv_tc launch (SPC_EXP_TRACE2 build, globaltimer ns):
entry, setup done, first stage full, last commit, exit; tiles / stages per CTA.

python -m paper_2511_20834_b200.build --exp TL -DSPC_EXP_TRACE2
SPC_LIB_OVERRIDE=paper_2511_20834_b200/exp_TL.so python scripts/timeline_conv.py --cin 64 --cout 64 --t -1 --n 18000
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("SPC_LIB_OVERRIDE", os.path.join(here, "..", "paper_2511_20834_b200", "exp_TL.so"))
import runpy
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
rel = (t[:5] - t0) / 1000.0
print(f"CTAs {n}: times in us from the first CTA entry")
for name, row in zip(["entry", "setup", "first_full", "last_commit", "exit"], rel):
    v = row[t[list(["entry", "setup", "first_full", "last_commit", "exit"]).index(name)] > 0] if False else row
    print(f"  {name:12s} min {v.min():7.2f}  median {np.median(v):7.2f}  max {v.max():7.2f}")
for nm, sl in (("last tfull seen", 5), ("last tile stored", 6), ("epilogue end", 7)):
    v = (t[sl] - t0) / 1000.0
    print(f"  {nm:14s} min {v.min():7.2f}  median {np.median(v):7.2f}  max {v.max():7.2f}")
busy = rel[3] - rel[2]
print(f"  first_full->last_commit  median {np.median(busy):.2f} max {busy.max():.2f};  setup->first_full median {np.median(rel[2]-rel[1]):.2f}")
ex = rel[4]
for b in np.argsort(-ex)[:6]:
    print(f"  slow CTA {b:4d}: " + " ".join(f"{nm}={rel[i][b]:7.2f}" for i, nm in enumerate(["entry", "setup", "first_full", "last_commit", "exit"])))
