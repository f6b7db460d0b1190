"""Build libspc.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a.

Usage: python -m paper_2511_20834_b200.build   (or __graft_entry__.build())
Experiments: python -m paper_2511_20834_b200.build --exp NAME -DMACRO ...  -> exp_NAME.so
(load it with SPC_LIB_OVERRIDE=.../exp_NAME.so)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspc.so")
SOURCES = ["spc_host.cu", "spc_sort.cu", "spc_kmap.cu", "spc_conv.cu", "spc_dense.cu", "spc_wgrad.cu"]
HEADERS = ["spc_common.cuh", "spc_ptx.cuh", "spc_tile.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "spc.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, exp: str | None = None, defines=()) -> str:
    lib = LIB if exp is None else os.path.join(HERE, f"exp_{exp}.so")
    if exp is None and not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build" if exp is None else f"build_{exp}")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p, src in zip(procs, SOURCES):
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
                           "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    exp = sys.argv[sys.argv.index("--exp") + 1] if "--exp" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, exp=exp,
                defines=[a for a in sys.argv[1:] if a.startswith("-D")]))
