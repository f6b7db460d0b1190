"""paper_2511_20834_b200 -- B200 (sm_100a) sparse-convolution hot path of Spira
(arXiv 2511.20834), behind the C ABI declared in include/spc.h.

This module is the thin Python binding: it only marshals torch tensors (device memory,
streams) into the C entry points of ``libspc.so`` -- every step of the hot path runs in
the library's CUDA kernels.  Function names follow the C ABI.  There is no CPU fallback:
if ``libspc.so`` is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspc.so")
_PRODUCT_LIB = LIB_PATH

SPC_OK = 0
SPC_F32, SPC_F16, SPC_BF16 = 0, 1, 2
SPC_T_ALL_OS = -1
SPC_T_ALL_WS = 0
SPC_KMAP_HALVE_SYMMETRIC = 0x1
SPC_KMAP_CHECK_SORTED = 0x2
SPC_KMAP_COUNT_SEARCHES = 0x4
SPC_KMAP_DENSITY_ORDER = 0x8
SPC_KMAP_SIMPLE_BSEARCH = 0x10
SPC_FLAG_RANGE, SPC_FLAG_DUPLICATE, SPC_FLAG_UNSORTED, SPC_FLAG_CAPACITY = 1, 2, 4, 8
SPC_MAX_KVOL = 125
# spc_option
SPC_OPT_CONV_TILE_ROWS, SPC_OPT_CONV_STAGE_KB, SPC_OPT_CONV_OS_SPLIT, SPC_OPT_CONV_SPLIT_MIN = 0, 1, 2, 3
SPC_OPT_CONV_CLAIM_AHEAD, SPC_OPT_CONV_DENSITY_ORDER, SPC_OPT_PDL, SPC_OPT_KMAP_POOL_KEYS = 4, 5, 6, 7
SPC_OPT_CONV_DENSE_CENTRE, SPC_OPT_CONV_CTA_PAIR, SPC_OPT_CONV_MAPS_READY, SPC_OPT_CONV_BULK_RED = 8, 9, 10, 11
SPC_OPT_WGRAD_ITEMS_PER_SM, SPC_OPT_CONV_SPLIT_TILES, SPC_OPT_CONV_MAX_CTAS = 12, 13, 14
SPC_OPT_CONV_BLK_KB = 15

_DT = {torch.float32: SPC_F32, torch.float16: SPC_F16, torch.bfloat16: SPC_BF16}
_TORCH_DT = {v: k for k, v in _DT.items()}


class SpcError(RuntimeError):
    pass


class PackSpec(ctypes.Structure):
    """spc_pack_spec: field widths (z least significant) and the headroom they were
    planned for (``reach`` per axis, ``out_stride``; reading A4)."""
    _fields_ = [("bits_b", ctypes.c_int32), ("bits_x", ctypes.c_int32), ("bits_y", ctypes.c_int32),
                ("bits_z", ctypes.c_int32), ("reach", ctypes.c_int32), ("out_stride", ctypes.c_int32)]

    def __init__(self, bits_b=0, bits_x=0, bits_y=0, bits_z=0, reach=0, out_stride=1):
        super().__init__(bits_b, bits_x, bits_y, bits_z, reach, out_stride)

    def used_bits(self) -> int:
        return self.bits_b + self.bits_x + self.bits_y + self.bits_z

    def astuple(self):
        """(bits_b, bits_x, bits_y, bits_z)"""
        return (self.bits_b, self.bits_x, self.bits_y, self.bits_z)

    def __repr__(self):
        return f"PackSpec{self.astuple()}(reach={self.reach}, out_stride={self.out_stride})"


class Geom(ctypes.Structure):
    """spc_geom.  ``kernel_size``: odd int K (Delta(K, s_p)) or a (Kx, Ky, Kz) box,
    even sizes {0..K-1} (reading E1)."""
    _fields_ = [("kernel_size", ctypes.c_int32), ("stride", ctypes.c_int32), ("dilation", ctypes.c_int32),
                ("tensor_stride", ctypes.c_int32), ("transposed", ctypes.c_int32),
                ("kernel_size_y", ctypes.c_int32), ("kernel_size_z", ctypes.c_int32)]

    def __init__(self, kernel_size=3, stride=1, dilation=1, tensor_stride=1, transposed=0):
        if isinstance(kernel_size, (tuple, list)):
            kx, ky, kz = (int(v) for v in kernel_size)
        else:
            kx = ky = kz = int(kernel_size)
        super().__init__(kx, stride, dilation, tensor_stride, int(transposed), ky, kz)

    def box(self):
        return (self.kernel_size, self.kernel_size_y or self.kernel_size, self.kernel_size_z or self.kernel_size)

    def k_vol(self):
        kx, ky, kz = self.box()
        return kx * ky * kz

    def key(self):
        return (self.kernel_size, self.stride, self.dilation, self.tensor_stride, self.transposed) + \
            ((self.box(),) if len(set(self.box())) > 1 else ())

    def __repr__(self):
        return "Geom(K=%s, s=%d, d=%d, ts=%d, tr=%d)" % ((self.box() if len(set(self.box())) > 1 else self.kernel_size,
                                                          self.stride, self.dilation, self.tensor_stride, self.transposed))


class _Kmap(ctypes.Structure):
    _fields_ = [("geom", Geom), ("t", ctypes.c_int32), ("k_vol", ctypes.c_int32), ("k_dense", ctypes.c_int32),
                ("n_lists", ctypes.c_int32), ("halved", ctypes.c_int32), ("key_bits", ctypes.c_int32),
                ("tile_words", ctypes.c_int32),
                ("n_in", ctypes.c_int64), ("n_out", ctypes.c_int64),
                ("n_in_dev", ctypes.c_void_p), ("n_out_dev", ctypes.c_void_p),
                ("in_keys", ctypes.c_void_p), ("out_keys", ctypes.c_void_p),
                ("os_table", ctypes.c_void_p), ("ws_pairs", ctypes.c_void_p), ("counts_dev", ctypes.c_void_p),
                ("tile_mask_dev", ctypes.c_void_p), ("search_stats_dev", ctypes.c_void_p),
                ("os_rows", ctypes.c_void_p), ("os_table_ord", ctypes.c_void_p), ("tile_mask_ord", ctypes.c_void_p),
                ("tile_order", ctypes.c_void_p),
                ("dense_k", ctypes.c_int16 * SPC_MAX_KVOL), ("list_k", ctypes.c_int16 * SPC_MAX_KVOL),
                ("list_mirror", ctypes.c_int8 * SPC_MAX_KVOL)]


class Epilogue(ctypes.Structure):
    """spc_epilogue: y = acc * scale + shift, + residual, then ReLU."""
    _fields_ = [("scale", ctypes.c_void_p), ("shift", ctypes.c_void_p), ("relu", ctypes.c_int32)]


SPC_WEIGHT_FORWARD, SPC_WEIGHT_DGRAD, SPC_WEIGHT_DGRAD_MIRROR = 0, 1, 2

_lib = None


def lib():
    """Load libspc.so (built by __graft_entry__.build() / paper_2511_20834_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SpcError(f"{LIB_PATH} not built: run python -m paper_2511_20834_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, U32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
        sig = {
            "spc_status_string": ([ctypes.c_int], ctypes.c_char_p),
            "spc_last_error_detail": ([], ctypes.c_char_p),
            "spc_version": ([], ctypes.c_int),
            "spc_kmap_struct_bytes": ([], SZ),
            "spc_set_option": ([I32, I64], ctypes.c_int),
            "spc_get_option": ([I32], I64),
            "spc_set_trace": ([P, I64], ctypes.c_int),
            "spc_trace_launch_desc": ([I32], ctypes.c_char_p),
            "spc_plan_pack": ([P, P, I32, I32, I32, ctypes.POINTER(PackSpec)], ctypes.c_int),
            "spc_pack_offset": ([PackSpec, I32, I32, I32], I64),
            "spc_downsample_mask": ([PackSpec, I32], ctypes.c_uint64),
            "spc_pack_sort_workspace_size": ([I64], SZ),
            "spc_pack_sort": ([P, I64, P, PackSpec, P, P, P, P, SZ, P], ctypes.c_int),
            "spc_pack_sort32": ([P, I64, P, PackSpec, P, P, P, P, SZ, P], ctypes.c_int),
            "spc_gather_rows": ([P, I64, P, I64, P, I32, P, I64, P], ctypes.c_int),
            "spc_regular_outputs_workspace_size": ([I64, Geom], SZ),
            "spc_regular_outputs": ([P, I64, P, PackSpec, Geom, P, P, P, SZ, P], ctypes.c_int),
            "spc_voxelize_workspace_size": ([I64], SZ),
            "spc_voxelize": ([P, I64, P, I64, P, P, PackSpec, P, I64, I32, P, P, P, P, I64, I32, P, P, P, SZ, P],
                             ctypes.c_int),
            "spc_downsample_workspace_size": ([I64, I32], SZ),
            "spc_downsample": ([P, I64, P, PackSpec, I32, P, P, P, P, SZ, P], ctypes.c_int),
            "spc_kmap_bytes": ([Geom, I32, U32, I64, I64], SZ),
            "spc_build_kmap": ([P, I64, P, P, I64, P, PackSpec, Geom, I32, U32, P, SZ, P,
                                ctypes.POINTER(_Kmap), P], ctypes.c_int),
            "spc_build_kmap32": ([P, I64, P, P, I64, P, PackSpec, Geom, I32, U32, P, SZ, P,
                                  ctypes.POINTER(_Kmap), P], ctypes.c_int),
            "spc_kmap_export": ([ctypes.POINTER(_Kmap), P, I64, ctypes.POINTER(I64), P], ctypes.c_int),
            "spc_prepared_weight_bytes": ([I32, I32, I32, I32], SZ),
            "spc_prepare_weight": ([P, I32, I32, I32, I32, P, P], ctypes.c_int),
            "spc_conv_workspace_size": ([ctypes.POINTER(_Kmap), I32, I32], SZ),
            "spc_conv_forward": ([ctypes.POINTER(_Kmap), P, I64, I32, I32, P, I32, P, I64, I32, P, I64, P, SZ, P],
                                 ctypes.c_int),
            "spc_conv_forward_ex": ([ctypes.POINTER(_Kmap), P, I64, I32, I32, P, I32, P, I64, I32, P, I64,
                                     ctypes.POINTER(Epilogue), P, SZ, P], ctypes.c_int),
            "spc_bn_fold": ([P, P, P, P, ctypes.c_float, I32, P, P, P], ctypes.c_int),
            "spc_prepare_weight_ex": ([P, I32, I32, I32, I32, I32, P, P], ctypes.c_int),
            "spc_add_rows": ([P, I64, P, I64, I64, P, I32, I32, I32, P], ctypes.c_int),
            "spc_conv_wgrad": ([ctypes.POINTER(_Kmap), P, I64, I32, I32, P, I64, I32, P, P], ctypes.c_int),
            "spc_network_workspace_size": ([I64, I32, P, P, P, I32], SZ),
            "spc_shard_ranges": ([P, I64, P, P, I64, P, PackSpec, Geom, I32, P, P], ctypes.c_int),
            "spc_network_kmaps": ([P, I64, P, PackSpec, I32, P, P, P, I32, P, P, P, P, P, SZ, P], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            if LIB_PATH != _PRODUCT_LIB and not hasattr(L, name):
                continue   # an older experiment build (scripts/ab_lib.py) may predate a symbol
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != SPC_OK:
        L = lib()
        raise SpcError(f"{what}: {L.spc_status_string(status).decode()}: {L.spc_last_error_detail().decode()}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _tstream(stream, device):
    """The torch stream the library call will be enqueued on."""
    return stream if stream is not None else torch.cuda.current_stream(device)


def _alloc(shape, dtype, device, stream, zero: bool = False) -> torch.Tensor:
    """A temporary the library fills on ``stream``: allocated (and zero-filled) ON that
    stream, so the caching allocator orders its reuse and the fill before the kernels that
    use it, whichever stream is current.  Callers that drop it before the
    stream has consumed it call ``_release(t, stream)``."""
    st = _tstream(stream, device)
    with torch.cuda.stream(st):
        return torch.zeros(shape, dtype=dtype, device=device) if zero else torch.empty(shape, dtype=dtype,
                                                                                       device=device)


def _release(t, stream):
    """Mark a temporary as in use on ``stream`` until the work enqueued so far completes."""
    if t is not None and t.is_cuda:
        t.record_stream(_tstream(stream, t.device))


def _ws(nbytes: int, device, zero: bool = False, stream=None) -> torch.Tensor:
    n = max(int(nbytes), 256)
    return _alloc((n,), torch.uint8, device, stream, zero)


def spc_set_option(option: int, value: int):
    """Process-wide performance option (spc.h spc_option); value < 0 restores the default."""
    _check(lib().spc_set_option(int(option), int(value)), "spc_set_option")


def spc_get_option(option: int) -> int:
    return int(lib().spc_get_option(int(option)))


def spc_set_trace(buf: torch.Tensor | None):
    """Device event trace of the feature kernels (spc.h): buf int64 [1 + 2*cap] (zero buf[0]
    before a traced pass), or None to turn tracing off."""
    cap = 0 if buf is None else (buf.numel() - 1) // 2
    _check(lib().spc_set_trace(_ptr(buf), cap), "spc_set_trace")


def spc_trace_records(buf: torch.Tensor):
    """[sync] -> numpy structured records (t_ns, launch, event, cta, aux) of a trace buffer."""
    h = buf.cpu().numpy().view(np.uint64)
    n = int(min(h[0], (h.size - 1) // 2))
    r = h[1:1 + 2 * n].reshape(n, 2)
    info = r[:, 1]
    out = np.zeros(n, dtype=[("t", np.int64), ("launch", np.int32), ("event", np.int32), ("cta", np.int32),
                             ("aux", np.int32)])
    out["t"] = r[:, 0].astype(np.int64)
    out["launch"] = (info >> np.uint64(48)).astype(np.int32)
    out["event"] = ((info >> np.uint64(40)) & np.uint64(0xff)).astype(np.int32)
    out["cta"] = ((info >> np.uint64(24)) & np.uint64(0xffff)).astype(np.int32)
    out["aux"] = (info & np.uint64(0xffffff)).astype(np.int32)
    return out


def spc_trace_launch_desc(launch: int) -> str:
    return lib().spc_trace_launch_desc(int(launch)).decode()


# ---------------------------------------------------------------------------------------
# A1/A2
# ---------------------------------------------------------------------------------------

def spc_plan_pack(lo, hi, n_batch: int = 1, max_out_stride: int = 1, max_reach: int = 0) -> PackSpec:
    spec = PackSpec()
    lo_a = (ctypes.c_int32 * 3)(*[int(v) for v in lo])
    hi_a = (ctypes.c_int32 * 3)(*[int(v) for v in hi])
    _check(lib().spc_plan_pack(lo_a, hi_a, int(n_batch), int(max_out_stride), int(max_reach), ctypes.byref(spec)),
           "spc_plan_pack")
    return spec


def spc_pack_offset(spec: PackSpec, dx: int, dy: int, dz: int) -> int:
    return int(lib().spc_pack_offset(spec, int(dx), int(dy), int(dz)))


def spc_downsample_mask(spec: PackSpec, m: int) -> int:
    return int(lib().spc_downsample_mask(spec, int(m)))


def spc_pack_sort(coords: torch.Tensor, spec: PackSpec, status: torch.Tensor | None = None, stream=None,
                  keys_out=None, perm_out=None, ws=None, n_dev=None, key_bits: int = 64):
    """coords int32 [n,4] (b,x,y,z) on the GPU -> (keys uint64-as-int64 [n], perm int32 [n], status uint32[1]).
    ``n_dev``: optional device int64 live row count (<= n); rows beyond it are ignored.
    ``key_bits=32``: uint32 keys (as int32) through spc_pack_sort32 (spec fields <= 32 bits)."""
    assert coords.is_cuda and coords.dtype == torch.int32 and coords.is_contiguous() and coords.shape[-1] == 4
    n = coords.shape[0]
    dev = coords.device
    keys = keys_out if keys_out is not None else _alloc(n, torch.int32 if key_bits == 32 else torch.int64, dev, stream)
    perm = perm_out if perm_out is not None else _alloc(n, torch.int32, dev, stream)
    if status is None:
        status = _alloc(1, torch.int32, dev, stream, zero=True)
    L = lib()
    wsb = int(L.spc_pack_sort_workspace_size(n))
    own_ws = ws is None or ws.numel() < wsb
    if own_ws:
        ws = _ws(wsb, dev, stream=stream)
    fn = L.spc_pack_sort32 if keys.dtype == torch.int32 else L.spc_pack_sort
    _check(fn(_ptr(coords), n, _ptr(n_dev), spec, _ptr(keys), _ptr(perm), _ptr(status), _ptr(ws), ws.numel(),
                           _stream(stream)), "spc_pack_sort")
    if own_ws:
        _release(ws, stream)
    return keys, perm, status


def spc_gather_rows(src: torch.Tensor, perm: torch.Tensor, out: torch.Tensor | None = None, n_dev=None,
                    stream=None) -> torch.Tensor:
    """out[r] = src[perm[r]] (rows of a 2-D tensor; row bytes multiple of 16)."""
    n = perm.shape[0]
    if out is None:
        out = _alloc((n,) + tuple(src.shape[1:]), src.dtype, src.device, stream)
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else out[0].numel() * out.element_size()
    _check(lib().spc_gather_rows(_ptr(src), src.stride(0) * src.element_size(), _ptr(perm), n, _ptr(n_dev),
                                 row_bytes, _ptr(out), out.stride(0) * out.element_size(), _stream(stream)),
           "spc_gather_rows")
    return out


# ---------------------------------------------------------------------------------------
# NEXT-3 spconv regular output sites
# ---------------------------------------------------------------------------------------

def spc_regular_outputs(keys: torch.Tensor, spec: PackSpec, geom: Geom, n_dev=None, stream=None):
    """Sorted unique output keys of spconv's regular rule for a forward layer of ``geom``
    (every stride-lattice site whose kernel box touches an input key).  Returns (out_keys
    int64 [n * k_vol] -- the first n_out valid --, n_out int64 [1] on the device)."""
    n = keys.shape[0]
    dev = keys.device
    out = _alloc(max(n * geom.k_vol(), 1), torch.int64, dev, stream)
    n_out = _alloc(1, torch.int64, dev, stream)
    L = lib()
    ws = _ws(int(L.spc_regular_outputs_workspace_size(n, geom)), dev, stream=stream)
    _check(L.spc_regular_outputs(_ptr(keys), n, _ptr(n_dev), spec, geom, _ptr(out), _ptr(n_out), _ptr(ws), ws.numel(),
                                 _stream(stream)), "spc_regular_outputs")
    _release(ws, stream)
    return out, n_out


# ---------------------------------------------------------------------------------------
# NEXT-2 voxelization front-end
# ---------------------------------------------------------------------------------------

def spc_voxelize(points: torch.Tensor, grid, spec: PackSpec, batch: torch.Tensor | None = None,
                 feats: torch.Tensor | None = None, out_dtype=torch.float32, n_dev=None, status=None, stream=None):
    """Raw points -> voxels (P:96 v = floor(p/g)): points float32 [n, >=3] (x, y, z
    first, row stride = points.stride(0)), grid (gx, gy, gz) metres, batch int32 [n] or None,
    feats float32 [n, c] or None.  Returns (keys int64 [n] -- the first n_vox are the sorted
    unique voxel keys --, n_vox int64 [1], point_voxel int32 [n], mean features [n, c] of
    out_dtype or None, status uint32[1], bad_point int64 [1] (-1 or the first non-finite point))."""
    assert points.is_cuda and points.dtype == torch.float32 and points.dim() == 2 and points.stride(1) == 1
    n = points.shape[0]
    dev = points.device
    c = 0 if feats is None else feats.shape[1]
    if feats is not None:
        assert feats.dtype == torch.float32 and feats.stride(1) == 1
    keys = _alloc(n, torch.int64, dev, stream)
    n_vox = _alloc(1, torch.int64, dev, stream)
    pv = _alloc(n, torch.int32, dev, stream)
    out = _alloc((n, c), out_dtype, dev, stream) if c else None
    if status is None:
        status = _alloc(1, torch.int32, dev, stream, zero=True)
    bad = _alloc(1, torch.int64, dev, stream)
    g = (ctypes.c_float * 3)(*[float(x) for x in grid])
    L = lib()
    ws = _ws(int(L.spc_voxelize_workspace_size(n)), dev, stream=stream)
    _check(L.spc_voxelize(_ptr(points), points.stride(0), _ptr(batch), n, _ptr(n_dev), g, spec, _ptr(feats),
                          feats.stride(0) if feats is not None else 0, c, _ptr(keys), _ptr(n_vox), _ptr(pv), _ptr(out),
                          out.stride(0) if out is not None else 0, _DT[out_dtype], _ptr(status), _ptr(bad), _ptr(ws),
                          ws.numel(), _stream(stream)), "spc_voxelize")
    _release(ws, stream)
    return keys, n_vox, pv, out, status, bad


# ---------------------------------------------------------------------------------------
# A3
# ---------------------------------------------------------------------------------------

def spc_downsample(keys: torch.Tensor, spec: PackSpec, log2_strides, n_dev=None, stream=None):
    """Sorted unique keys -> (level_keys int64 [L, n] (row l valid up to level_n[l]), level_n int64 [L])."""
    n = keys.shape[0]
    L_ = len(log2_strides)
    dev = keys.device
    out = _alloc((L_, n), torch.int64, dev, stream)
    level_n = _alloc(L_, torch.int64, dev, stream)
    m = (ctypes.c_int32 * L_)(*[int(v) for v in log2_strides])
    L = lib()
    ws = _ws(L.spc_downsample_workspace_size(n, L_), dev, stream=stream)
    _check(L.spc_downsample(_ptr(keys), n, _ptr(n_dev), spec, L_, m, _ptr(out), _ptr(level_n), _ptr(ws), ws.numel(),
                            _stream(stream)), "spc_downsample")
    _release(ws, stream)
    return out, level_n


# ---------------------------------------------------------------------------------------
# A4-A8
# ---------------------------------------------------------------------------------------

class KernelMap:
    """A built kernel map: the C struct plus the torch buffer that owns its memory."""

    def __init__(self, struct: _Kmap, buf: torch.Tensor, keepalive=()):
        self.c = struct
        self.buf = buf
        self._keep = keepalive

    @property
    def k_dense(self):
        return self.c.k_dense

    @property
    def n_lists(self):
        return self.c.n_lists

    @property
    def k_vol(self):
        return self.c.k_vol

    @property
    def n_out(self):
        return self.c.n_out

    @property
    def dense_k(self):
        return [self.c.dense_k[i] for i in range(self.c.k_dense)]

    @property
    def list_k(self):
        return [self.c.list_k[i] for i in range(self.c.n_lists)]

    def _view(self, ptr, count, dtype):
        off = ptr - self.buf.data_ptr()
        es = torch.empty((), dtype=dtype).element_size()
        return self.buf[off:off + count * es].view(dtype)

    def os_table(self) -> torch.Tensor:
        return self._view(self.c.os_table, self.c.n_out * self.c.k_dense, torch.int32).view(self.c.n_out,
                                                                                              self.c.k_dense)

    def tile_mask(self) -> torch.Tensor:
        """[tiles, words] int32: bit c of a 128-row tile set iff dense column c has a match in it."""
        n, w = self.c.n_out, self.c.tile_words
        tiles = (n + 127) // 128
        return self._view(self.c.tile_mask_dev, tiles * w, torch.int32).view(tiles, w)

    def density_order(self):
        """(os_rows [n_out], os_table_ord [n_out, k_dense], tile_mask_ord [tiles, words]) of a
        map built with SPC_KMAP_DENSITY_ORDER, else None (views of the map buffer)."""
        if not self.c.os_rows:
            return None
        n, kd, w = self.c.n_out, self.c.k_dense, self.c.tile_words
        tiles = (n + 127) // 128
        return (self._view(self.c.os_rows, n, torch.int32),
                self._view(self.c.os_table_ord, n * kd, torch.int32).view(n, kd),
                self._view(self.c.tile_mask_ord, tiles * w, torch.int32).view(tiles, w))

    def tile_order(self):
        """Heaviest-first OS tile orders of a density-ordered map, else None:
        (order128 [ceil(n/128)], order256 [ceil(n/256)], weight128, weight256) over the
        capacity n_out (spc.h: 128-row tiles by descending popcount of their ordered tile
        mask, then 256-row tiles likewise; then the weights in those two orders)."""
        if not self.c.tile_order:
            return None
        t128 = (self.c.n_out + 127) // 128
        t256 = (self.c.n_out + 255) // 256
        v = self._view(self.c.tile_order, 4 * t128, torch.int32).view(4, t128)
        return v[0], v[1, :t256], v[2], v[3, :t256]

    def counts(self) -> torch.Tensor:
        return self._view(self.c.counts_dev, 2 * SPC_MAX_KVOL, torch.int32)

    def search_stats(self) -> torch.Tensor | None:
        if not self.c.search_stats_dev:
            return None
        return self._view(self.c.search_stats_dev, 2, torch.int64)

    def ws_pairs(self, l: int) -> torch.Tensor:
        cnt = int(self.counts()[SPC_MAX_KVOL + l].item())
        base = self.c.ws_pairs + l * self.c.n_out * 8
        return self._view(base, 2 * cnt, torch.int32).view(cnt, 2)


def spc_kmap_bytes(geom: Geom, t: int, flags: int, n_in: int, n_out: int) -> int:
    return int(lib().spc_kmap_bytes(geom, int(t), int(flags), int(n_in), int(n_out)))


def spc_build_kmap(in_keys: torch.Tensor, out_keys: torch.Tensor, spec: PackSpec, geom: Geom,
                   t: int = SPC_T_ALL_OS, flags: int = 0, n_in_dev=None, n_out_dev=None, status=None,
                   stream=None, buf: torch.Tensor | None = None) -> KernelMap:
    """``buf``: optional pre-allocated uint8 buffer (>= spc_kmap_bytes + 256 bytes), so a
    build can be re-issued (and graph-captured) without allocating."""
    n_in, n_out = in_keys.shape[0], out_keys.shape[0]
    nbytes = spc_kmap_bytes(geom, t, flags, n_in, n_out)
    if nbytes == 0:
        raise SpcError(f"spc_kmap_bytes: unsupported geometry {geom!r}")
    if buf is None or buf.numel() < nbytes + 256:
        buf = _alloc(nbytes + 256, torch.uint8, in_keys.device, stream)
    off = (-buf.data_ptr()) % 256
    buf = buf[off:off + nbytes]
    km = _Kmap()
    fn = lib().spc_build_kmap32 if in_keys.dtype == torch.int32 else lib().spc_build_kmap
    _check(fn(_ptr(in_keys), n_in, _ptr(n_in_dev), _ptr(out_keys), n_out, _ptr(n_out_dev), spec,
                                geom, int(t), int(flags), _ptr(buf), nbytes, _ptr(status), ctypes.byref(km),
                                _stream(stream)), "spc_build_kmap")
    return KernelMap(km, buf, (in_keys, out_keys, n_in_dev, n_out_dev))


def spc_kmap_export(km: KernelMap, stream=None) -> np.ndarray:
    """[sync] -> int32 [nnz, 3] (k, out, in) triples, lexicographically sorted."""
    L = lib()
    nnz = ctypes.c_int64(0)
    _check(L.spc_kmap_export(ctypes.byref(km.c), None, 0, ctypes.byref(nnz), _stream(stream)), "spc_kmap_export")
    out = np.empty((nnz.value, 3), dtype=np.int32)
    _check(L.spc_kmap_export(ctypes.byref(km.c), out.ctypes.data_as(ctypes.c_void_p), nnz.value, ctypes.byref(nnz),
                             _stream(stream)), "spc_kmap_export")
    return out


# ---------------------------------------------------------------------------------------
# A9-A12
# ---------------------------------------------------------------------------------------

def spc_prepare_weight(weight: torch.Tensor, stream=None) -> torch.Tensor:
    """weight [K^3, C_in, C_out] (f32/f16/bf16, on the GPU) -> prepared weight for spc_conv_forward."""
    kv, ci, co = weight.shape
    w = weight.contiguous()
    dt = _DT[w.dtype]
    out = _alloc(w.numel(), w.dtype, w.device, stream)
    _check(lib().spc_prepare_weight(_ptr(w), kv, ci, co, dt, _ptr(out), _stream(stream)), "spc_prepare_weight")
    return out


def spc_prepare_weight_ex(weight: torch.Tensor, mode: int, stream=None) -> torch.Tensor:
    """weight [K^3, C_in, C_out] of a FORWARD layer -> prepared weight of mode SPC_WEIGHT_*
    (DGRAD: W_k^T, DGRAD_MIRROR: W_{K^3-1-k}^T, i.e. a (K^3, C_out -> C_in) layer)."""
    kv, ci, co = weight.shape
    w = weight.contiguous()
    out = _alloc(w.numel(), w.dtype, w.device, stream)
    _check(lib().spc_prepare_weight_ex(_ptr(w), kv, ci, co, _DT[w.dtype], int(mode), _ptr(out), _stream(stream)),
           "spc_prepare_weight_ex")
    return out


def spc_bn_fold(gamma, beta, mean, var, eps: float, stream=None):
    """Inference batch norm folded on the device -> (scale, shift) fp32 [c]."""
    c = gamma.numel()
    scale = _alloc(c, torch.float32, gamma.device, stream)
    shift = _alloc(c, torch.float32, gamma.device, stream)
    _check(lib().spc_bn_fold(_ptr(gamma), _ptr(beta), _ptr(mean), _ptr(var), float(eps), c, _ptr(scale), _ptr(shift),
                             _stream(stream)), "spc_bn_fold")
    return scale, shift


def spc_conv_wgrad(km: KernelMap, f_in: torch.Tensor, d_out: torch.Tensor, c_in: int, c_out: int,
                   d_weight: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """dW [K^3, c_in, c_out] fp32 += the weight gradient of Eq. (2) over the map's pairs."""
    if d_weight is None:
        d_weight = _alloc((km.c.k_vol, c_in, c_out), torch.float32, f_in.device, stream, zero=True)
    _check(lib().spc_conv_wgrad(ctypes.byref(km.c), _ptr(f_in), f_in.stride(0), _DT[f_in.dtype], int(c_in),
                                _ptr(d_out), d_out.stride(0), int(c_out), _ptr(d_weight), _stream(stream)),
           "spc_conv_wgrad")
    return d_weight


def spc_add_rows(dst: torch.Tensor, src: torch.Tensor, n_dev=None, stream=None, accumulate: bool = True):
    """dst[:n] += src[:n] (or = src[:n] when not accumulate; row slices with their own
    strides; n = *n_dev or dst rows)."""
    _check(lib().spc_add_rows(_ptr(dst), dst.stride(0), _ptr(src), src.stride(0), dst.shape[0], _ptr(n_dev),
                              dst.shape[1], _DT[dst.dtype], int(bool(accumulate)), _stream(stream)), "spc_add_rows")
    return dst


def spc_conv_workspace_size(km: KernelMap, c_out: int, out_dtype=torch.float32) -> int:
    return int(lib().spc_conv_workspace_size(ctypes.byref(km.c), int(c_out), _DT[out_dtype]))


def spc_conv_forward(km: KernelMap, f_in: torch.Tensor, weight_prepared: torch.Tensor, c_in: int, c_out: int,
                     out: torch.Tensor | None = None, out_dtype=None, residual: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None, stream=None, scale: torch.Tensor | None = None,
                     shift: torch.Tensor | None = None, relu: bool = False) -> torch.Tensor:
    """Eq. (2) for the map ``km``: f_in [n_in, >=c_in] (row stride = f_in.stride(0)) -> out [n_out, c_out].
    ``ws``: byte tensor of >= spc_conv_workspace_size bytes, all-zero before its first use
    (torch.zeros); every call leaves it all-zero again."""
    out_dtype = out_dtype or (out.dtype if out is not None else f_in.dtype)
    if out is None:
        out = _alloc((km.n_out, c_out), out_dtype, f_in.device, stream)
    need = spc_conv_workspace_size(km, c_out, out_dtype)
    own_ws = ws is None
    if own_ws:
        ws = _ws(need, f_in.device, zero=True, stream=stream)   # all-zero on first use (spc.h), filled on `stream`
    elif ws.numel() < need:
        raise ValueError(f"spc_conv_forward: ws has {ws.numel()} bytes, needs {need}")
    if scale is None and shift is None and not relu:
        _check(lib().spc_conv_forward(ctypes.byref(km.c), _ptr(f_in), f_in.stride(0), _DT[f_in.dtype], int(c_in),
                                      _ptr(weight_prepared), int(c_out), _ptr(out), out.stride(0), _DT[out.dtype],
                                      _ptr(residual), residual.stride(0) if residual is not None else 0, _ptr(ws),
                                      ws.numel(), _stream(stream)), "spc_conv_forward")
    else:
        epi = Epilogue(scale.data_ptr() if scale is not None else None,
                       shift.data_ptr() if shift is not None else None, int(bool(relu)))
        _check(lib().spc_conv_forward_ex(ctypes.byref(km.c), _ptr(f_in), f_in.stride(0), _DT[f_in.dtype], int(c_in),
                                         _ptr(weight_prepared), int(c_out), _ptr(out), out.stride(0), _DT[out.dtype],
                                         _ptr(residual), residual.stride(0) if residual is not None else 0,
                                         ctypes.byref(epi), _ptr(ws), ws.numel(), _stream(stream)),
               "spc_conv_forward_ex")
    if own_ws:
        _release(ws, stream)
    return out


# ---------------------------------------------------------------------------------------
# A13
# ---------------------------------------------------------------------------------------

class NetworkIndex:
    """Pre-allocated state of spc_network_kmaps for one (n0, n_levels, map list): the
    workspace, the level key / count buffers and the C kmap structs.  ``run()`` only
    enqueues work (no allocation), so it can be captured in a CUDA graph."""

    def __init__(self, n0: int, spec: PackSpec, n_levels: int, geoms, ts, flags=None, device="cuda"):
        self.n0, self.spec, self.n_levels = int(n0), spec, int(n_levels)
        n = len(geoms)
        self.n = n
        self.G = (Geom * max(n, 1))(*geoms)
        self.T = (ctypes.c_int32 * max(n, 1))(*[int(t) for t in ts])
        self.F = (ctypes.c_uint32 * max(n, 1))(*[int(f) for f in (flags or [0] * n)])
        need = int(lib().spc_network_workspace_size(self.n0, self.n_levels, self.G, self.T, self.F, n))
        ws = torch.empty(need + 256, dtype=torch.uint8, device=device)
        off = (-ws.data_ptr()) % 256
        self._ws_full = ws
        self.ws = ws[off:off + need]
        self.level_keys = torch.empty((self.n_levels, self.n0), dtype=torch.int64, device=device)
        self.level_n = torch.empty(self.n_levels, dtype=torch.int64, device=device)
        self.structs = (_Kmap * max(n, 1))()
        self.maps = [None] * n

    def run(self, v0_keys: torch.Tensor, n0_dev=None, status=None, stream=None):
        _check(lib().spc_network_kmaps(_ptr(v0_keys), self.n0, _ptr(n0_dev), self.spec, self.n_levels, self.G, self.T,
                                       self.F, self.n, _ptr(self.level_keys), _ptr(self.level_n), self.structs,
                                       _ptr(status), _ptr(self.ws), self.ws.numel(), _stream(stream)),
               "spc_network_kmaps")
        if self.maps[0] is None or self.n == 0:
            self.maps = [KernelMap(self.structs[i], self.ws, (v0_keys, self.level_keys, self.level_n))
                         for i in range(self.n)]
        return self.maps


def spc_network_kmaps(v0_keys: torch.Tensor, spec: PackSpec, n_levels: int, geoms, ts, flags=None, n0_dev=None,
                      status=None, stream=None):
    """Network-wide indexing -> (level_keys [n_levels, n0], level_n [n_levels], [KernelMap per entry])."""
    ni = NetworkIndex(v0_keys.shape[0], spec, n_levels, geoms, ts, flags, device=v0_keys.device)
    maps = ni.run(v0_keys, n0_dev=n0_dev, status=status, stream=stream)
    for m in maps:
        m._keep = m._keep + (ni,)
    return ni.level_keys, ni.level_n, maps


# ---------------------------------------------------------------------------------------
# multi-GPU, one large scene: output ranges + input halos
# ---------------------------------------------------------------------------------------

def spc_shard_ranges(in_keys: torch.Tensor, out_keys: torch.Tensor, spec: PackSpec, geom: Geom, n_shards: int,
                     n_in_dev=None, n_out_dev=None, stream=None) -> torch.Tensor:
    """-> device int64 [n_shards, 4]: (out_lo, out_hi, in_lo, in_hi) per shard (spc.h)."""
    b = _alloc((int(n_shards), 4), torch.int64, in_keys.device, stream)
    _check(lib().spc_shard_ranges(_ptr(in_keys), in_keys.shape[0], _ptr(n_in_dev), _ptr(out_keys), out_keys.shape[0],
                                  _ptr(n_out_dev), spec, geom, int(n_shards), _ptr(b), _stream(stream)),
           "spc_shard_ranges")
    return b

