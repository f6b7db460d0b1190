"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every entry
point include/spc.h declares, host-side helpers behave, and the binding's struct
layouts match the C structs."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2511_20834_b200 as spc
from paper_2511_20834_b200 import build as spc_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    spc_build.build()
    return spc.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "spc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spc_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("spc_pack_sort", "spc_build_kmap", "spc_conv_forward", "spc_network_kmaps"):
        assert n in names


def test_every_declared_symbol_is_exported(L):
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing


def test_struct_layout_matches(L):
    assert L.spc_kmap_struct_bytes() == ctypes.sizeof(spc._Kmap)


def test_status_strings(L):
    assert L.spc_status_string(0) == b"SPC_OK"
    assert L.spc_status_string(3) == b"SPC_ERR_RANGE"


def test_plan_pack_and_helpers(L):
    # KITTI-like extents (+-1024 voxels in x/y at 0.05 m, z -80..48), strides up to 16, reach 16
    s = spc.spc_plan_pack((-1024, -1024, -80), (1023, 1023, 48), n_batch=1, max_out_stride=16, max_reach=16)
    assert s.astuple() == (0, 12, 12, 8)
    s8 = spc.spc_plan_pack((-1024, -1024, -80), (1023, 1023, 48), n_batch=8, max_out_stride=16, max_reach=16)
    assert s8.bits_b == 3
    assert spc.spc_pack_offset(s, -1, -1, -1) == -((1 << 20) + (1 << 8) + 1)
    m1 = spc.spc_downsample_mask(s, 1)
    assert m1 == ((1 << 32) - 1) & ~((1 << 0) | (1 << 8) | (1 << 20))
    with pytest.raises(spc.SpcError):
        spc.spc_plan_pack((-(1 << 30),) * 3, ((1 << 30),) * 3)


def test_kmap_bytes_and_errors(L):
    g = spc.Geom(3, 1, 1, 1, 0)
    assert spc.spc_kmap_bytes(g, -1, 0, 1000, 1000) >= 1000 * 27 * 4
    # NEXT-3 boxes: K = 2 ({0, 1}^3) and (3, 1, 1) are planned; sizes outside 1..5 are not
    assert spc.spc_kmap_bytes(spc.Geom(2, 2, 1, 1, 0), -1, 0, 10, 10) >= 10 * 8 * 4
    assert spc.spc_kmap_bytes(spc.Geom((3, 1, 1), 1, 1, 1, 0), -1, 0, 10, 10) >= 10 * 3 * 4
    assert spc.spc_kmap_bytes(spc.Geom(6, 1, 1, 1, 0), -1, 0, 10, 10) == 0
    assert spc.spc_kmap_bytes(spc.Geom((3, 0, 7), 1, 1, 1, 0), -1, 0, 10, 10) == 0


def test_plan_records_headroom(L):
    s = spc.spc_plan_pack((-1024, -1024, -80), (1023, 1023, 48), n_batch=1, max_out_stride=16, max_reach=16)
    assert (s.reach, s.out_stride) == (16, 16)


def _build_kmap_status(L, spec, geom):
    """spc_build_kmap's host-side checks only (no keys, no device work): returns the status."""
    km = spc._Kmap()
    nbytes = spc.spc_kmap_bytes(geom, -1, 0, 0, 0)
    return L.spc_build_kmap(None, 0, None, None, 0, None, spec, geom, -1, 0, ctypes.c_void_p(1 << 20),
                            nbytes, None, ctypes.byref(km), None)


def test_build_kmap_refuses_reach_beyond_plan(L):
    """Reading A4 / S:84: a map reaching further than the planned headroom is an
    error (SPC_ERR_RANGE), never a silent carry into the neighbouring field."""
    spec = spc.spc_plan_pack((-100, -100, -20), (100, 100, 20), 1, max_out_stride=4, max_reach=2)
    # within the plan: past the host checks (without a GPU the enqueue itself then fails)
    assert _build_kmap_status(L, spec, spc.Geom(3, 1, 1, 2, 0)) != 3          # r*ts*d = 2
    assert _build_kmap_status(L, spec, spc.Geom(5, 1, 1, 1, 0)) != 3          # r = 2
    assert _build_kmap_status(L, spec, spc.Geom(3, 1, 2, 2, 0)) == 3          # 1*2*2 = 4 > 2
    assert _build_kmap_status(L, spec, spc.Geom(5, 1, 1, 2, 0)) == 3          # 2*2 = 4 > 2
    assert _build_kmap_status(L, spec, spc.Geom(3, 2, 1, 4, 0)) == 3          # coarse stride 8 > 4
    assert b"reach" in L.spc_last_error_detail() or b"stride" in L.spc_last_error_detail()


def test_options_roundtrip(L):
    assert spc.spc_get_option(spc.SPC_OPT_CONV_STAGE_KB) == 72
    spc.spc_set_option(spc.SPC_OPT_CONV_STAGE_KB, 48)
    assert spc.spc_get_option(spc.SPC_OPT_CONV_STAGE_KB) == 48
    spc.spc_set_option(spc.SPC_OPT_CONV_STAGE_KB, -1)
    assert spc.spc_get_option(spc.SPC_OPT_CONV_STAGE_KB) == 72
    with pytest.raises(spc.SpcError):
        spc.spc_set_option(99, 1)


def test_no_environment_knobs_in_the_product():
    """The product library reads no environment variables (tuning is explicit through
    spc_set_option) and carries no experiment-only code paths."""
    csrc = os.path.join(ROOT, "paper_2511_20834_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert "getenv" not in src, f
        assert "SPC_EXP_" not in src, f
