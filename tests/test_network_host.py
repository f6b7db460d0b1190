"""Host logic of network.py on CPU (no GPU): the layer lists, the training buffer versioning
(ssa_buffers), the backward's first-touch plan, and the pipeline split points."""
import pytest

import bench
from paper_2511_20834_b200 import network as nw


class _Net:
    """Just the attributes the host-side helpers read."""

    def __init__(self, layers, widths, out_name):
        self.layers, self.out_name = layers, out_name
        self.gbufs = {k: _Shape(w) for k, w in widths.items()}
        self._plan = None


class _Shape:
    def __init__(self, w):
        self.shape = (1, w)


def _lists():
    L, w = nw.minkunet42_layers(3)
    yield "minkunet42", L, w, "out"
    L, w = nw.minkunet42_layers(2)
    yield "minkunet42_k2", L, w, "out"
    L, w, out = nw.second_backbone_layers(5)
    yield "secondk5", L, w, out


@pytest.mark.parametrize("name,layers,widths,out", list(_lists()))
def test_layer_lists(name, layers, widths, out):
    if name.startswith("minkunet42"):
        assert sum(s.map_key[0] > 1 for s in layers) == 42 and sum(s.map_key[0] == 1 for s in layers) == 7
    else:
        assert len(layers) == 20 and sum(s.map_key[1] == 2 for s in layers) == 3   # 17 subm + 3 strided
    for s in layers:   # every write fits its buffer
        assert s.dst_col + s.c_out <= widths[s.dst]


@pytest.mark.parametrize("name,layers,widths,out", list(_lists()))
def test_ssa_buffers_never_overwrite(name, layers, widths, out):
    """After versioning, no layer writes a column range another layer already wrote, and
    every read names the latest version written before it (or an input buffer)."""
    L, w2 = nw.ssa_buffers(layers, widths)
    written = {}
    for s in L:
        for a, b in written.get(s.dst, []):
            assert s.dst_col + s.c_out <= a or b <= s.dst_col, s.name
        written.setdefault(s.dst, []).append((s.dst_col, s.dst_col + s.c_out))
        assert s.dst in w2
    # reads refer to buffers that exist and were written earlier (or the input x0)
    seen = {"x0"}
    for s in L:
        assert s.src in seen, s.name
        if s.residual:
            assert s.residual[0] in seen, s.name
        seen.add(s.dst)


@pytest.mark.parametrize("name,layers,widths,out", list(_lists()))
def test_first_touch_plan(name, layers, widths, out):
    """The backward's plan: no gradient buffer needs a zero fill for these networks, every
    gradient region read by the backward is fully written before it is read, and each
    region's first contribution is the one that overwrites."""
    L, w2 = nw.ssa_buffers(layers, widths)
    out_name = [s.dst for s in L if s.dst.split("@")[0] == out][-1]
    net = _Net(L, w2, out_name)
    plan = nw.SparseNet._first_touch(net)
    assert plan["zero"] == []
    cover = {out_name: [(0, w2[out_name])]}
    for i in reversed(range(len(L))):
        s = L[i]
        segs = sorted(cover.get(s.dst, []))
        at = s.dst_col
        for a, b in segs:
            if a <= at:
                at = max(at, b)
        assert at >= s.dst_col + s.c_out, (s.name, "read before written")
        for key, region in (("res", (s.residual[0], s.residual[1], s.residual[1] + s.c_out) if s.residual else None),
                            ("dgrad", (s.src, s.src_col, s.src_col + s.c_in) if i > 0 else None)):
            if region is None:
                continue
            b_, lo, hi = region
            first = not any(a < hi and lo < b for a, b in cover.get(b_, []))
            assert plan[key][i] == first, (s.name, key)
            cover.setdefault(b_, []).append((lo, hi))


def test_pipeline_split_points():
    L, _ = nw.minkunet42_layers(3)
    net = _Net(L, {}, "out")
    assert nw.pipeline_index_after(net) == [s.name for s in L].index("enc4.down")
    assert bench.pipeline_split(net) == 22
    L2, _, _ = nw.second_backbone_layers(5)
    net2 = _Net(L2, {}, "out")
    assert nw.pipeline_index_after(net2) == -1   # the deepest level is the network's tail
    assert bench.pipeline_split(net2) == 9


class _GeomNet:
    def __init__(self, keys, lo, hi):
        self.map_keys, self.t = keys, {k: 4 for k in keys}
        self.density_order, self.order_min_ts, self.order_max_ts = True, lo, hi


@pytest.mark.parametrize("lo,hi", [(0, 1 << 30), (2, 1 << 30), (0, 2), (4, 8)])
def test_map_flags_follow_the_order_window(lo, hi):
    """Per-map build flags: halving on submanifold K > 1 maps, the density order exactly on
    the forward maps whose fine tensor stride lies in [order_min_ts, order_max_ts]."""
    from paper_2511_20834_b200 import SPC_KMAP_DENSITY_ORDER, SPC_KMAP_HALVE_SYMMETRIC
    L, _ = nw.minkunet42_layers(3)
    keys = list(dict.fromkeys(s.map_key for s in L))
    _, _, flags = nw.SparseNet._geoms(_GeomNet(keys, lo, hi))
    for mk, f in zip(keys, flags):
        K, stride, tsd, tr = mk
        assert bool(f & SPC_KMAP_HALVE_SYMMETRIC) == (stride == 1 and K > 1), mk
        assert bool(f & SPC_KMAP_DENSITY_ORDER) == (lo <= tsd <= hi), mk
