"""Timeline of one k_conv_tc launch (CTA 0) from the SPC_EXP_TRACE build (experiments)."""
import ctypes, os, sys
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("SPC_LIB_OVERRIDE", os.path.join(here, "..", "paper_2511_20834_b200", "exp_TRACE.so"))
import runpy
sys.argv = ["probe_conv.py"] + sys.argv[1:] + ["--reps", "1"]
runpy.run_path(os.path.join(here, "probe_conv.py"), run_name="__main__")
import paper_2511_20834_b200 as spc
L = spc.lib()
buf = np.zeros((8, 4096), np.int64)
L.spc_exp_trace_read.argtypes = [ctypes.c_void_p]
L.spc_exp_trace_read(buf.ctypes.data)
names = {2: "mma_full", 4: "fenced", 5: "issued", 3: "committed", 6: "epi_tfull", 7: "epi_done"}
t0 = buf[buf > 0].min()
for i in range(0, 40):
    print(i, " ".join(f"{n}={(buf[k, i] - t0) if buf[k, i] else -1:8d}" for k, n in names.items()))
for k, n in names.items():
    v = buf[k][buf[k] > 0]
    if len(v) > 2:
        print(n, "count", len(v), "median delta", np.median(np.diff(v)))
