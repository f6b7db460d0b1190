"""CPU oracle for the Spira SpC hot path (arXiv 2511.20834) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product path
(``paper_2511_20834_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``spc_oracle.c``); this module only marshals numpy
arrays through ctypes.  Every function follows a definition in PAPER.md:

=====================  =============================================================
``sort_coords``        canonical lexicographic order (§5.2)
``pack``               A1 biased-field key (§5.3 + DESIGN.md readings A3/A5)
``downsample``         Eq. (1) V_q = floor(V_p/s_q)*s_q, unique (§2.1)
``offsets``            Delta(K, s_p) lexicographic, dz fastest
``kmap``               M[i,k] = j iff p_j = q_i + delta_k, hash-set lookup
``conv``               Eq. (2) in fp64, OS or WS loop order
``conv_rows``          Eq. (2) for sampled output rows (full-size sampled parity)
``offsets/kmap/conv``  also over (Kx, Ky, Kz) boxes, even sizes {0..K-1}
``regular_outputs``    spconv's regular output rule
``voxelize``           v = floor(p/g) in float32, unique, mean feature (§2.1)
=====================  =============================================================

Parity pins: tests/test_oracle_pins.py (brute force, closed forms, paper examples,
torch conv3d in float64).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spc_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_LIB_OMP_PATH = os.path.join(_HERE, "liboracle_omp.so")
_lib = None
_use_omp = False


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: liboracle.so (plain C11, -O2, single-threaded, what the
    parity tests use) and liboracle_omp.so (the same source with -fopenmp: Eq. (2) output
    rows spread over the host cores, for timing the CPU baseline)."""
    dep = max(os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "spc_oracle.h")))
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < dep:
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", _SRC, "-o", _LIB_PATH, "-lm"])
    if force or not os.path.exists(_LIB_OMP_PATH) or os.path.getmtime(_LIB_OMP_PATH) < dep:
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", _SRC, "-o", _LIB_OMP_PATH, "-lm"])
    return _LIB_PATH


def use_openmp(on: bool = True):
    """Route later calls to the OpenMP build (bench.py's cpu_baseline / reference arm)."""
    global _use_omp, _lib
    if bool(on) != _use_omp:
        _use_omp = bool(on)
        _lib = None


def num_threads() -> int:
    return int(_L().orc_num_threads())


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_OMP_PATH if _use_omp else _LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        lib.orc_sort_coords.argtypes = [P, I64, P, P]
        lib.orc_sort_coords.restype = I64
        lib.orc_pack.argtypes = [P, I64, I, I, I, I, P]
        lib.orc_pack.restype = I64
        lib.orc_round_down.argtypes = [ctypes.c_int32, ctypes.c_int32]
        lib.orc_round_down.restype = ctypes.c_int32
        lib.orc_downsample.argtypes = [P, I64, ctypes.c_int32, P]
        lib.orc_downsample.restype = I64
        lib.orc_offsets.argtypes = [I, I, P, P]
        lib.orc_offsets.restype = I
        lib.orc_kmap.argtypes = [P, I64, P, I64, I, I, I, P, I64]
        lib.orc_kmap.restype = I64
        lib.orc_conv.argtypes = [P, I64, P, I64, I, I, I, P, I, P, I, P, I]
        lib.orc_conv.restype = I64
        lib.orc_conv_rows.argtypes = [P, I64, P, P, I64, I, I, I, P, I, P, I, P]
        lib.orc_conv_rows.restype = I64
        lib.orc_offsets3.argtypes = [I, I, I, I, P, P]
        lib.orc_offsets3.restype = I
        lib.orc_kmap3.argtypes = [P, I64, P, I64, I, I, I, I, I, P, I64]
        lib.orc_kmap3.restype = I64
        lib.orc_conv3.argtypes = [P, I64, P, I64, I, I, I, I, I, P, I, P, I, P, I]
        lib.orc_conv3.restype = I64
        lib.orc_conv_rows3.argtypes = [P, I64, P, P, I64, I, I, I, I, I, P, I, P, I, P]
        lib.orc_conv_rows3.restype = I64
        lib.orc_regular_outputs.argtypes = [P, I64, I, I, I, I, I, P]
        lib.orc_regular_outputs.restype = I64
        lib.orc_voxelize.argtypes = [P, I64, P, I64, P, P, I64, I, P, P, P]
        lib.orc_voxelize.restype = I64
        lib.orc_conv_dgrad3.argtypes = [P, I64, P, I64, I, I, I, I, I, P, I, P, I, P]
        lib.orc_conv_dgrad3.restype = I64
        lib.orc_conv_dgrad_rows3.argtypes = [P, I64, P, I64, P, I64, I, I, I, I, I, P, I, P, I, P]
        lib.orc_conv_dgrad_rows3.restype = I64
        lib.orc_conv_wgrad3.argtypes = [P, I64, P, I64, I, I, I, I, I, P, I, P, I, P]
        lib.orc_conv_wgrad3.restype = I64
        lib.orc_bn_relu.argtypes = [P, I64, I, P, P, P, P, ctypes.c_double, P, I, P]
        lib.orc_bn_relu.restype = None
        lib.orc_num_threads.argtypes = []
        lib.orc_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def sort_coords(coords):
    """-> (sorted int32 [n,4], perm int32 [n] with sorted[p] = coords[perm[p]], n_dups)."""
    c = _c(coords, np.int32).reshape(-1, 4)
    n = c.shape[0]
    s = np.empty_like(c)
    perm = np.empty(n, np.int32)
    d = _L().orc_sort_coords(_p(c), n, _p(s), _p(perm))
    return s, perm, int(d)


def pack(coords, bits):
    """bits = (Bb, Bx, By, Bz) -> (uint64 keys [n], n_out_of_range)."""
    c = _c(coords, np.int32).reshape(-1, 4)
    keys = np.empty(c.shape[0], np.uint64)
    bad = _L().orc_pack(_p(c), c.shape[0], int(bits[0]), int(bits[1]), int(bits[2]), int(bits[3]),
                        _p(keys))
    return keys, int(bad)


def round_down(v: int, s: int) -> int:
    return int(_L().orc_round_down(int(v), int(s)))


def downsample(coords, s: int):
    """Eq. (1): sorted unique int32 [m, 4]."""
    c = _c(coords, np.int32).reshape(-1, 4)
    out = np.empty_like(c)
    m = _L().orc_downsample(_p(c), c.shape[0], int(s), _p(out))
    if m < 0:
        raise ValueError("orc_downsample failed")
    return out[:m].copy()


def _box(K):
    """K (odd, cubic: Delta(K, s_p) of P:111) or a tuple (Kx, Ky, Kz) (the generalised
    box of SURVEY NEXT-3, even sizes {0..K-1}) -> (kx, ky, kz, generalised?)."""
    if isinstance(K, (tuple, list)):
        return int(K[0]), int(K[1]), int(K[2]), True
    K = int(K)
    return K, K, K, K % 2 == 0


def offsets(K, spacing: int = 1):
    """-> (int32 [kv, 3] offsets, int32 [kv] L1 norm in units of ``spacing``).  An int K must
    be odd; a tuple (Kx, Ky, Kz) gives the generalised box (NEXT-3, reading E1)."""
    if not isinstance(K, (tuple, list)):
        kv = int(K) ** 3
        off = np.empty((max(kv, 1), 3), np.int32)
        l1 = np.empty(max(kv, 1), np.int32)
        r = _L().orc_offsets(int(K), int(spacing), _p(off), _p(l1))
        if r < 0:
            raise ValueError("even or non-positive K")
        return off, l1
    kx, ky, kz, _ = _box(K)
    kv = kx * ky * kz
    off = np.empty((max(kv, 1), 3), np.int32)
    l1 = np.empty(max(kv, 1), np.int32)
    if _L().orc_offsets3(kx, ky, kz, int(spacing), _p(off), _p(l1)) < 0:
        raise ValueError("non-positive kernel size")
    return off, l1


def kmap(in_coords, out_coords, K, spacing: int, transposed: bool = False):
    """-> int32 [nnz, 3] triples (k, out_index, in_index), lexicographically sorted.
    K: odd int or (Kx, Ky, Kz) (NEXT-3)."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    b = _c(out_coords, np.int32).reshape(-1, 4)
    L = _L()
    kx, ky, kz, gen = _box(K)

    def run(t, cap):
        if gen:
            return L.orc_kmap3(_p(a), a.shape[0], _p(b), b.shape[0], kx, ky, kz, int(spacing), int(transposed), t, cap)
        return L.orc_kmap(_p(a), a.shape[0], _p(b), b.shape[0], kx, int(spacing), int(transposed), t, cap)

    nnz = run(None, 0)
    if nnz < 0:
        raise ValueError("orc_kmap failed")
    t = np.empty((max(nnz, 1), 3), np.int32)
    run(_p(t), nnz)
    return t[:nnz]


def conv(in_coords, out_coords, K, spacing: int, F_in, W, transposed: bool = False,
         order: str = "os"):
    """Eq. (2) in fp64.  F_in [n_in, c_in], W [kv, c_in, c_out] -> F_out [n_out, c_out]."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    b = _c(out_coords, np.int32).reshape(-1, 4)
    F = _c(F_in, np.float64)
    Wd = _c(W, np.float64)
    c_in, c_out = Wd.shape[1], Wd.shape[2]
    kx, ky, kz, gen = _box(K)
    assert F.shape == (a.shape[0], c_in) and Wd.shape[0] == kx * ky * kz
    out = np.empty((b.shape[0], c_out), np.float64)
    o = 0 if order == "os" else 1
    if gen:
        r = _L().orc_conv3(_p(a), a.shape[0], _p(b), b.shape[0], kx, ky, kz, int(spacing), int(transposed),
                           _p(F), c_in, _p(Wd), c_out, _p(out), o)
    else:
        r = _L().orc_conv(_p(a), a.shape[0], _p(b), b.shape[0], kx, int(spacing), int(transposed),
                          _p(F), c_in, _p(Wd), c_out, _p(out), o)
    if r < 0:
        raise ValueError("orc_conv failed")
    return out


def conv_rows(in_coords, out_coords, rows, K, spacing: int, F_in, W, transposed: bool = False):
    """Eq. (2) for output rows ``rows`` only -> [len(rows), c_out] fp64."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    b = _c(out_coords, np.int32).reshape(-1, 4)
    rr = _c(rows, np.int64)
    F = _c(F_in, np.float64)
    Wd = _c(W, np.float64)
    c_in, c_out = Wd.shape[1], Wd.shape[2]
    kx, ky, kz, gen = _box(K)
    out = np.empty((rr.shape[0], c_out), np.float64)
    if gen:
        r = _L().orc_conv_rows3(_p(a), a.shape[0], _p(b), _p(rr), rr.shape[0], kx, ky, kz, int(spacing),
                                int(transposed), _p(F), c_in, _p(Wd), c_out, _p(out))
    else:
        r = _L().orc_conv_rows(_p(a), a.shape[0], _p(b), _p(rr), rr.shape[0], kx, int(spacing),
                               int(transposed), _p(F), c_in, _p(Wd), c_out, _p(out))
    if r < 0:
        raise ValueError("orc_conv_rows failed")
    return out


def regular_outputs(in_coords, K, spacing: int, out_stride: int):
    """spconv's regular output rule: sorted unique int32 [m, 4] sites
    (b, p - delta) on the out_stride lattice, p in in_coords, delta in the offset box."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    kx, ky, kz, _ = _box(K)
    out = np.empty((max(a.shape[0] * kx * ky * kz, 1), 4), np.int32)
    m = _L().orc_regular_outputs(_p(a), a.shape[0], kx, ky, kz, int(spacing), int(out_stride), _p(out))
    if m < 0:
        raise ValueError("orc_regular_outputs failed")
    return out[:m].copy()


def voxelize(points, grid, batch=None, feats=None):
    """Voxelization: points float32 [n, >=3] (x, y, z first),
    grid (gx, gy, gz), batch int32 [n] or None, feats float32 [n, c] or None.
    -> (coords int32 [V, 4] canonical (b, x, y, z), point_voxel int32 [n],
        mean fp64 [V, c] or None).  ValueError names the first non-finite point."""
    P = np.ascontiguousarray(points, dtype=np.float32)
    n, ld = P.shape
    g = _c(grid, np.float32).reshape(3)
    b = None if batch is None else _c(batch, np.int32).reshape(n)
    F = None if feats is None else _c(feats, np.float32).reshape(n, -1)
    c = 0 if F is None else F.shape[1]
    coords = np.empty((max(n, 1), 4), np.int32)
    pv = np.empty(max(n, 1), np.int32)
    mean = np.empty((max(n, 1), max(c, 1)), np.float64) if F is not None else None
    nv = _L().orc_voxelize(_p(P), ld, _p(b) if b is not None else None, n, _p(g),
                           _p(F) if F is not None else None, c, c, _p(coords), _p(pv),
                           _p(mean) if mean is not None else None)
    if nv < 0:
        raise ValueError(f"voxelize: point {-nv - 1} is not finite (or its quotient leaves int32)")
    return coords[:nv], pv[:n], (mean[:nv, :c] if mean is not None else None)


# ---------------------------------------------------------------------------------------
# training path (gradients of Eq. (2)) and the fused BN / residual / ReLU
# epilogue -- see spc_oracle.h for the definitions each function writes out.
# ---------------------------------------------------------------------------------------

def conv_dgrad(in_coords, out_coords, K, spacing: int, dF_out, W, transposed: bool = False):
    """d(Eq. 2)/d f_in: dF_in [n_in, c_in] fp64 from dF_out [n_out, c_out], W [kv, c_in, c_out]."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    b = _c(out_coords, np.int32).reshape(-1, 4)
    G = _c(dF_out, np.float64)
    Wd = _c(W, np.float64)
    c_in, c_out = Wd.shape[1], Wd.shape[2]
    kx, ky, kz, _ = _box(K)
    assert G.shape == (b.shape[0], c_out) and Wd.shape[0] == kx * ky * kz
    out = np.empty((a.shape[0], c_in), np.float64)
    r = _L().orc_conv_dgrad3(_p(a), a.shape[0], _p(b), b.shape[0], kx, ky, kz, int(spacing), int(transposed),
                             _p(G), c_out, _p(Wd), c_in, _p(out))
    if r < 0:
        raise ValueError("orc_conv_dgrad3 failed")
    return out


def conv_dgrad_rows(in_coords, out_coords, rows, K, spacing: int, dF_out, W, transposed: bool = False):
    """dF_in for input rows ``rows`` only, by gathering over the output set -> [len(rows), c_in]."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    b = _c(out_coords, np.int32).reshape(-1, 4)
    rr = _c(rows, np.int64)
    G = _c(dF_out, np.float64)
    Wd = _c(W, np.float64)
    c_in, c_out = Wd.shape[1], Wd.shape[2]
    kx, ky, kz, _ = _box(K)
    out = np.empty((rr.shape[0], c_in), np.float64)
    r = _L().orc_conv_dgrad_rows3(_p(a), a.shape[0], _p(b), b.shape[0], _p(rr), rr.shape[0], kx, ky, kz,
                                  int(spacing), int(transposed), _p(G), c_out, _p(Wd), c_in, _p(out))
    if r < 0:
        raise ValueError("orc_conv_dgrad_rows3 failed")
    return out


def conv_wgrad(in_coords, out_coords, K, spacing: int, F_in, dF_out, transposed: bool = False):
    """d(Eq. 2)/d W: dW [kv, c_in, c_out] fp64 from F_in [n_in, c_in] and dF_out [n_out, c_out]."""
    a = _c(in_coords, np.int32).reshape(-1, 4)
    b = _c(out_coords, np.int32).reshape(-1, 4)
    F = _c(F_in, np.float64)
    G = _c(dF_out, np.float64)
    c_in, c_out = F.shape[1], G.shape[1]
    kx, ky, kz, _ = _box(K)
    assert F.shape[0] == a.shape[0] and G.shape[0] == b.shape[0]
    out = np.empty((kx * ky * kz, c_in, c_out), np.float64)
    r = _L().orc_conv_wgrad3(_p(a), a.shape[0], _p(b), b.shape[0], kx, ky, kz, int(spacing), int(transposed),
                             _p(F), c_in, _p(G), c_out, _p(out))
    if r < 0:
        raise ValueError("orc_conv_wgrad3 failed")
    return out


def bn_relu(x, gamma=None, beta=None, mean=None, var=None, eps: float = 1e-5, residual=None, relu: bool = True):
    """relu(bn(x) + residual) per channel (inference BN), fp64; gamma None: no normalisation."""
    X = _c(x, np.float64)
    n, c = X.shape
    y = np.empty_like(X)
    prm = [None if v is None else _c(v, np.float64).reshape(c) for v in (gamma, beta, mean, var)]
    if prm[0] is not None:
        assert all(v is not None for v in prm)
    R = None if residual is None else _c(residual, np.float64).reshape(n, c)
    _L().orc_bn_relu(_p(X), n, c, *[(_p(v) if v is not None else None) for v in prm], float(eps),
                     _p(R) if R is not None else None, int(bool(relu)), _p(y))
    return y
