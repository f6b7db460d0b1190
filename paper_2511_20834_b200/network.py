"""MinkUNet-42 (C2/C4) and a SECOND/CenterPoint-style K=5 backbone (C3) over libspc.

``SparseNet`` runs any layer list (``ConvSpec``) built by ``minkunet42_layers()`` or
``second_backbone_layers()``; ``SparseUNet`` is the MinkUNet-42 instance.

Orchestration only: every step of a forward pass is a C-ABI call of libspc (pack+sort,
row gather, network-wide kernel maps, 49 sparse convolutions with fused residual adds).
BN/ReLU are identity (out of scope); weights are seeded random bf16.
Channel-concatenation skips are free: encoder outputs are written straight into a
column slice of the decoder's concat buffer (ld_out > c_out).

Layer list (public MinkowskiEngine/TorchSparse MinkUNet with K=3 down/up;
``net="minkunet42_k2"``: TorchSparse's K=2 stride-2 down/up):
cs = [32, 32, 64, 128, 256, 256, 128, 96, 96]; stem 2 x SubM K3; 4 encoder stages
(Down K3 s2 + 2 ResBlocks); 4 decoder stages (Up K3 s2 transposed + concat + 2
ResBlocks) = 42 layers with K = 3 plus 7 1x1 projections.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

import paper_2511_20834_b200 as spc

CS = [32, 32, 64, 128, 256, 256, 128, 96, 96]
C_IN_RAW = 4
C_IN_PAD = 16   # tcgen05 kind::f16 needs K multiple of 16; the extra input channels are 0


@dataclasses.dataclass
class ConvSpec:
    name: str
    map_key: tuple          # (K, stride, tensor_stride, transposed)
    c_in: int
    c_out: int
    src: str                # activation buffer read
    src_col: int            # first column read
    dst: str                # activation buffer written
    dst_col: int
    level_out: int
    residual: tuple | None = None   # (buffer, first column) added to the output
    c_in_flops: int = 0     # channels counted for algorithmic FLOPs (stem: 4 real channels)


def minkunet42_layers(down_k: int = 3):
    """down_k = 3: the paper's odd-K reading (A10); down_k = 2: TorchSparse's MinkUNet
    down / up layers (K = 2, stride 2, offsets {0, s_p}^3)."""
    L = []
    lvl_buf = {}

    def conv(name, mk, ci, co, src, sc, dst, dc, lo, res=None, ci_fl=None):
        L.append(ConvSpec(name, mk, ci, co, src, sc, dst, dc, lo, res, ci_fl or ci))

    def subm(l):
        return (3, 1, 2 ** l, 0)

    def one(l):
        return (1, 1, 2 ** l, 0)

    def resblock(tag, l, src, sc, ci, co, dst, dc):
        conv(f"{tag}.conv1", subm(l), ci, co, src, sc, f"h{l}", 0, l)
        if ci != co:
            conv(f"{tag}.proj", one(l), ci, co, src, sc, f"p{l}", 0, l)
            res = (f"p{l}", 0)
        else:
            res = (src, sc)
        conv(f"{tag}.conv2", subm(l), co, co, f"h{l}", 0, dst, dc, l, res)

    # decoder concat widths per level: up channels + skip channels
    up_c = {3: CS[5], 2: CS[6], 1: CS[7], 0: CS[8]}
    skip_c = {3: CS[3], 2: CS[2], 1: CS[1], 0: CS[0]}
    cat_w = {l: up_c[l] + skip_c[l] for l in up_c}

    # stem (level 0)
    conv("stem.conv1", subm(0), C_IN_PAD, CS[0], "x0", 0, "h0", 0, 0, None, C_IN_RAW)
    conv("stem.conv2", subm(0), CS[0], CS[0], "h0", 0, "cat0", up_c[0], 0)
    src, sc, ch = "cat0", up_c[0], CS[0]
    # encoder
    for i in range(1, 5):
        l = i
        conv(f"enc{i}.down", (down_k, 2, 2 ** (l - 1), 0), ch, ch, src, sc, f"d{l}", 0, l)
        dst, dc = (f"cat{l}", up_c[l]) if l < 4 else ("e4", 0)
        resblock(f"enc{i}.rb1", l, f"d{l}", 0, ch, CS[i], f"y{l}", 0)
        resblock(f"enc{i}.rb2", l, f"y{l}", 0, CS[i], CS[i], dst, dc)
        src, sc, ch = dst, dc, CS[i]
    # decoder
    for j in range(1, 5):
        l = 4 - j
        co = CS[4 + j]
        conv(f"dec{j}.up", (down_k, 2, 2 ** l, 1), ch, co, src, sc, f"cat{l}", 0, l)
        resblock(f"dec{j}.rb1", l, f"cat{l}", 0, cat_w[l], co, f"y{l}", 0)
        dst = "out" if l == 0 else f"z{l}"
        resblock(f"dec{j}.rb2", l, f"y{l}", 0, co, co, dst, 0)
        src, sc, ch = dst, 0, co
    widths = {"x0": C_IN_PAD, "out": CS[8], "e4": CS[4]}
    for l in range(4):
        widths[f"cat{l}"] = cat_w[l]
    for s in L:
        widths[s.dst] = max(widths.get(s.dst, 0), s.dst_col + s.c_out)
    return L, widths


def second_backbone_layers(K: int = 5, c_in_raw: int = 5):
    """C3: CenterPoint/SECOND-style sparse backbone (ResNL): stem SubM K3
    c_in -> 16; 4 stages (16/32/64/128 channels) of 4 SubM K-conv layers (2 residual blocks);
    3 strided K3 s2 downsamplings -> 20 SpC layers (17 submanifold + 3 strided)."""
    L = []
    chans = [16, 32, 64, 128]

    def conv(name, mk, ci, co, src, dst, lo, res=None, ci_fl=None):
        L.append(ConvSpec(name, mk, ci, co, src, 0, dst, 0, lo, res, ci_fl or ci))

    conv("stem", (3, 1, 1, 0), C_IN_PAD, chans[0], "x0", "a0", 0, None, c_in_raw)
    cur = "a0"
    for st, ch in enumerate(chans):
        l = st
        if st > 0:
            conv(f"down{st}", (3, 2, 2 ** (l - 1), 0), chans[st - 1], ch, cur, f"a{l}", l)
            cur = f"a{l}"
        for blk in range(2):
            conv(f"s{st}.b{blk}.conv1", (K, 1, 2 ** l, 0), ch, ch, cur, f"h{l}", l)
            nxt = f"b{l}" if cur != f"b{l}" else f"a{l}"
            conv(f"s{st}.b{blk}.conv2", (K, 1, 2 ** l, 0), ch, ch, f"h{l}", nxt, l, (cur, 0))
            cur = nxt
    widths = {"x0": C_IN_PAD}
    for s_ in L:
        widths[s_.dst] = max(widths.get(s_.dst, 0), s_.dst_col + s_.c_out)
    widths["out"] = chans[-1]
    return L, widths, cur


def ssa_buffers(layers, widths):
    """Training: the forward list reuses buffers (h{l}, y{l}, p{l} at every
    block of a level), but the weight gradient of layer i needs layer i's own input.  Give
    every write that overlaps an earlier write of the same buffer a fresh version (reads and
    residuals follow the latest version); disjoint column slices of one buffer -- the
    decoder's concat of up-sampled features and the encoder skip -- stay one buffer."""
    ver, written, out, w2 = {}, {}, [], dict(widths)

    def cur(b):
        return b if ver.get(b, 0) == 0 else f"{b}@{ver[b]}"

    for s in layers:
        src = cur(s.src)
        res = (cur(s.residual[0]), s.residual[1]) if s.residual else None
        d = cur(s.dst)
        lo, hi = s.dst_col, s.dst_col + s.c_out
        if any(lo < b and a < hi for a, b in written.get(d, [])):
            ver[s.dst] = ver.get(s.dst, 0) + 1
            d = cur(s.dst)
            w2[d] = widths[s.dst]
        written.setdefault(d, []).append((lo, hi))
        out.append(dataclasses.replace(s, src=src, dst=d, residual=res))
    return out, w2


def dgrad_map_key(map_key):
    """The map the data gradient of a layer runs on (spc.h, spc_prepare_weight_ex): a
    submanifold layer's own map (mirrored weights), else the map of the opposite
    direction (strided <-> transposed, same K and fine tensor stride)."""
    K, stride, ts, tr = map_key
    return map_key if stride == 1 else (K, stride, ts, 1 - tr)


def wgrad_map_key(map_key):
    """The map the weight gradient runs on: the same geometry with every offset weight-
    stationary (t = 0; halved for submanifold maps), i.e. compact pair lists -- an OS
    table would make the pair contraction walk every sentinel row."""
    if map_key[0] == 1:
        return map_key   # a K = 1 map has no sentinels (its only offset always matches)
    return tuple(map_key) + ("ws",)


def default_t(map_key):
    """Dataflow threshold per map before tuning (reading: the paper's UNet uses WS in most
    layers).  K=1 maps are always dense."""
    K, stride, ts, tr = map_key
    if K == 1:
        return spc.SPC_T_ALL_OS
    if stride == 1:
        return 2                       # hybrid: centre + 6 face neighbours dense
    return spc.SPC_T_ALL_OS


class SparseNet:
    """Forward pass of a sparse-conv layer list over libspc; every buffer pre-allocated for
    capacity n0 (all levels), so a pass is a fixed launch sequence (CUDA-graph capturable)."""

    def __init__(self, n0_cap: int, spec: spc.PackSpec, device="cuda", seed: int = 20834, t_override=None,
                 nnz_per_out: float = 10.0, net: str = "minkunet42", density_order: bool = True,
                 train: bool = False):
        self.dev = torch.device(device)
        self.density_order = bool(density_order)
        self.order_max_ts = 1 << 30   # density-order only maps whose fine tensor stride is <= this
        self.order_min_ts = 0         # ... and >= this
        self.early_maps = True   # layers >= 1 start their tile decode during the previous layer
        self.overlap_proj = True   # ResBlock 1x1 projections on a side stream beside conv1 (+1.7% C2)
        self.overlap_wgrad = True  # backward: weight gradients on a side stream beside the data gradients
        self.spec = spec
        self.n0 = int(n0_cap)
        if net in ("minkunet42", "minkunet42_k2"):
            self.layers, widths = minkunet42_layers(2 if net.endswith("_k2") else 3)
            self.out_name, self.n_levels = "out", 5
        elif net.startswith("second"):
            K = 5 if net.endswith("k5") else 3
            self.layers, widths, self.out_name = second_backbone_layers(K)
            self.n_levels = 4
        else:
            raise ValueError(net)
        self.train = bool(train)
        if self.train:
            self.layers, widths = ssa_buffers(self.layers, widths)
            self.out_name = [s.dst for s in self.layers if s.dst.split("@")[0] == self.out_name][-1]
        self.map_keys = []
        # forward maps first: a network build orders (SPC_KMAP_DENSITY_ORDER) the maps of its
        # first grouped launch, and the training maps only add to a second one
        keys = [s.map_key for s in self.layers]
        if self.train:
            keys += [dgrad_map_key(s.map_key) for s in self.layers] + [wgrad_map_key(s.map_key) for s in self.layers]
        for mk in keys:
            if mk not in self.map_keys:
                self.map_keys.append(mk)
        self.t = {mk: (t_override or {}).get(mk, default_t(mk)) for mk in self.map_keys if len(mk) == 4}
        # weights: seeded, bf16, prepared for the tcgen05 layout
        g = torch.Generator().manual_seed(seed)
        self.weights, self.raw_weights, self.dgrad_weights = [], [], []
        for s in self.layers:
            kv = s.map_key[0] ** 3
            a = math.sqrt(3.0 / (min(kv, nnz_per_out) * s.c_in_flops))
            w = (torch.rand(kv, s.c_in, s.c_out, generator=g) * 2 - 1) * a
            if s.c_in != s.c_in_flops:
                w[:, s.c_in_flops:, :] = 0
            wd = w.to(self.dev, torch.bfloat16)
            self.weights.append(spc.spc_prepare_weight(wd))
            if self.train:
                self.raw_weights.append(wd)
                self.dgrad_weights.append(spc.spc_prepare_weight_ex(
                    wd, spc.SPC_WEIGHT_DGRAD_MIRROR if s.map_key[1] == 1 else spc.SPC_WEIGHT_DGRAD))
        # activations (capacity n0 rows for every level)
        self.bufs = {name: torch.zeros(self.n0, w, dtype=torch.bfloat16, device=self.dev) for name, w in widths.items()}
        if self.train:   # gradient buffers (same layout as the activations) and fp32 dW per layer
            self.gbufs = {name: torch.zeros_like(b) for name, b in self.bufs.items()}
            self.dW = [torch.zeros(s.map_key[0] ** 3, s.c_in, s.c_out, dtype=torch.float32, device=self.dev)
                       for s in self.layers]
        self.coords_ws = None
        self.keys = torch.empty(self.n0, dtype=torch.int64, device=self.dev)
        self.perm = torch.empty(self.n0, dtype=torch.int32, device=self.dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.n_live = torch.zeros(1, dtype=torch.int64, device=self.dev)   # live voxel count (scans < n0)
        self.sort_ws = torch.empty(int(spc.lib().spc_pack_sort_workspace_size(self.n0)), dtype=torch.uint8,
                                   device=self.dev)
        self.conv_ws = None      # sized from spc_conv_workspace_size once the maps exist (index())
        self.netidx = None
        self.maps = None

    # ---------------------------------------------------------------------------------
    def _geoms(self):
        geoms, ts, flags = [], [], []
        for mk in self.map_keys:
            K, stride, tsd, tr = mk[:4]
            geoms.append(spc.Geom(K, stride, 1, tsd, tr))
            t = self.t[mk] if len(mk) == 4 else 0   # wgrad maps: all weight-stationary
            ts.append(t)
            f = spc.SPC_KMAP_HALVE_SYMMETRIC if (stride == 1 and K > 1) else 0
            if self.density_order and len(mk) == 4 and self.order_min_ts <= tsd <= self.order_max_ts:
                f |= spc.SPC_KMAP_DENSITY_ORDER      # OS part only; ignored when t leaves no OS part
            flags.append(f)
        return geoms, ts, flags

    def index(self, stream=None, n_dev=None):
        """Network-wide voxel indexing: all levels, then all maps.  ``n_dev``: device
        int64 live voxel count when the scan is smaller than the capacity n0."""
        if self.netidx is None:
            geoms, ts, flags = self._geoms()
            self.netidx = spc.NetworkIndex(self.n0, self.spec, self.n_levels, geoms, ts, flags, device=self.dev)
        kms = self.netidx.run(self.keys, n0_dev=n_dev, status=self.status, stream=stream)
        self.level_keys, self.level_n = self.netidx.level_keys, self.netidx.level_n
        self.maps = dict(zip(self.map_keys, kms))
        need = max(spc.spc_conv_workspace_size(self.maps[s.map_key], s.c_out) for s in self.layers)
        if self.train:   # the data gradients write n_in x c_in through the dgrad maps
            need = max([need] + [spc.spc_conv_workspace_size(self.maps[dgrad_map_key(s.map_key)], s.c_in)
                                 for s in self.layers])
        if self.conv_ws is None or self.conv_ws.numel() < need:
            # zero once (spc.h ws contract), on the stream the convolutions run on
            self.conv_ws = spc._ws(need, self.dev, zero=True, stream=stream)

    def set_t(self, t_map: dict):
        self.t.update(t_map)
        self.netidx = None

    def conv(self, i, stream=None):
        s = self.layers[i]
        km = self.maps[s.map_key]
        src = self.bufs[s.src][:, s.src_col:s.src_col + s.c_in]
        dst = self.bufs[s.dst][:, s.dst_col:s.dst_col + s.c_out]
        res = None
        if s.residual is not None:
            rb, rc = s.residual
            res = self.bufs[rb][:, rc:rc + s.c_out]
        spc.spc_conv_forward(km, src, self.weights[i], s.c_in, s.c_out, out=dst, residual=res, ws=self.conv_ws,
                             stream=stream)

    def forward(self, coords: torch.Tensor, feats: torch.Tensor, stream=None, n_live=None) -> torch.Tensor:
        """coords int32 [n,4] (any order), feats bf16 [n, 16] (first 4 channels real) -> out
        [n0, 96] whose first n rows are the scan's voxels in sorted (canonical) order.

        Any scan size n <= n0 (the capacity) runs on the same buffers: the live count
        travels on the device (``n_live``, int64 [1]; filled from n when omitted), so
        a CUDA graph captured once replays for every scan size when the caller pads
        coords / feats to n0 rows and writes the live count into ``n_live``."""
        n = coords.shape[0]
        if n > self.n0:
            raise ValueError(f"scan of {n} voxels exceeds the capacity {self.n0}")
        if n_live is None and n < self.n0:
            n_live = self.n_live
            st = stream if stream is not None else torch.cuda.current_stream(self.dev)
            with torch.cuda.stream(st):
                n_live.fill_(n)
        self.index_stage(coords, feats, stream, n_live)
        return self.conv_stage(stream)

    def _side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.dev)
        return self._side

    def index_stage(self, coords: torch.Tensor, feats: torch.Tensor, stream=None, n_live=None):
        """The voxel-indexing half of forward(): pack + sort, feature row gather, every
        level and every kernel map (n_live: as in forward, already filled)."""
        n = coords.shape[0]
        spc.spc_pack_sort(coords, self.spec, status=self.status, keys_out=self.keys[:n], perm_out=self.perm[:n],
                          ws=self.sort_ws, stream=stream, n_dev=n_live)
        spc.spc_gather_rows(feats, self.perm[:n], out=self.bufs["x0"][:n], n_dev=n_live, stream=stream)
        self.index(stream, n_dev=n_live)

    def conv_stage(self, stream=None, marks=None, start: int = 0, stop: int | None = None) -> torch.Tensor:
        """The feature-computation half of forward(): layers [start, stop) (default all) on
        the maps of the last index_stage().  marks: {layer index: event} recorded on
        `stream` after that layer."""
        side = self._side_stream() if self.overlap_proj else None
        st = stream if stream is not None else torch.cuda.current_stream(self.dev)
        pending = {}    # layer index -> event of a 1x1 projection running on the side stream
        issued = set()  # projections already issued on the side stream
        stop = len(self.layers) if stop is None else stop
        try:
            for i in range(start, stop):
                s = self.layers[i]
                if i in issued:
                    continue
                if side is not None and i + 2 < stop:
                    nx = self.layers[i + 1]
                    if nx.map_key[0] == 1 and nx.src == s.src and nx.src_col == s.src_col:
                        # a ResBlock's 1x1 projection reads the block input like conv1: run it on
                        # the side stream beside conv1; conv2 (its residual reader) waits for it
                        fork = torch.cuda.Event()
                        fork.record(st)
                        side.wait_event(fork)
                        with torch.cuda.stream(side):
                            spc.spc_set_option(spc.SPC_OPT_CONV_MAPS_READY, 0)
                            self.conv(i + 1, side)
                        done = torch.cuda.Event()
                        done.record(side)
                        pending[i + 2] = done
                        issued.add(i + 1)
                if i in pending:
                    st.wait_event(pending.pop(i))
                # after the first layer the maps and weights are long complete when the
                # preceding kernel starts: let each layer decode tiles early (PDL)
                spc.spc_set_option(spc.SPC_OPT_CONV_MAPS_READY, 1 if (i > start and self.early_maps) else 0)
                self.conv(i, stream)
                if marks and i in marks:
                    marks[i].record(stream)
        finally:
            spc.spc_set_option(spc.SPC_OPT_CONV_MAPS_READY, 0)
        return self.bufs[self.out_name]

    def backward(self, grad_out: torch.Tensor | None = None, stream=None):
        """Training: the backward pass of the last forward.  grad_out: bf16
        gradient of the output buffer (None: already in gbufs[out_name]).  Every layer in
        reverse order: wgrad (spc_conv_wgrad into self.dW[i], zeroed first), the residual
        branch (spc_add_rows), and the data gradient through the forward kernels on the
        dgrad map (spc_conv_forward accumulating into the source gradient through its
        residual operand).  The stem's input gradient is not formed.  Returns self.dW."""
        if not self.train:
            raise ValueError("SparseNet(train=True) is required for backward()")
        st = stream if stream is not None else torch.cuda.current_stream(self.dev)
        plan = self._first_touch()
        with torch.cuda.stream(st):
            for name in plan["zero"]:
                if name != self.out_name or grad_out is not None:
                    self.gbufs[name].zero_()
            for w in self.dW:
                w.zero_()
            if grad_out is not None:
                self.gbufs[self.out_name][: grad_out.shape[0]].copy_(grad_out)
        side = self._side_stream() if self.overlap_wgrad else None
        for i in reversed(range(len(self.layers))):
            if side is not None:
                # layer i's output gradient is final here (every reader came later in the
                # forward, so earlier here) and nothing in the backward writes it again: its
                # weight gradient runs on the side stream beside the data gradients
                ready = torch.cuda.Event()
                ready.record(st)
                side.wait_event(ready)
                with torch.cuda.stream(side):
                    self.backward_layer(i, side, parts=("wgrad",))
                self.backward_layer(i, stream, parts=("residual", "dgrad"))
            else:
                self.backward_layer(i, stream)
        if side is not None:
            done = torch.cuda.Event()
            done.record(side)
            st.wait_event(done)
        return self.dW

    def _first_touch(self):
        """Which gradient writes are the first to their region (they overwrite; later ones
        accumulate), so the gradient buffers need no zero fill: regions are column slices of
        a buffer; a buffer whose regions are read before fully written, or written partly
        over an earlier region, is zeroed and accumulated into instead.  Static per layer
        list (computed once)."""
        if getattr(self, "_plan", None) is not None:
            return self._plan
        zero = set()
        for attempt in range(2):
            written = {self.out_name: [(0, self.gbufs[self.out_name].shape[1])]}
            first_res, first_dgrad = {}, {}

            def covered(name, lo, hi):
                segs = sorted(written.get(name, []))
                at = lo
                for a, b in segs:
                    if a > at:
                        break
                    at = max(at, b)
                return at >= hi

            def write(name, lo, hi):
                segs = written.setdefault(name, [])
                if name in zero:
                    segs.append((lo, hi))
                    return False
                overlap = [s for s in segs if s[0] < hi and lo < s[1]]
                if not overlap:
                    segs.append((lo, hi))
                    return True
                if not covered(name, lo, hi):
                    zero.add(name)   # partial overlap: zero the buffer, accumulate everywhere
                segs.append((lo, hi))
                return False

            for i in reversed(range(len(self.layers))):
                s = self.layers[i]
                if s.dst not in zero and not covered(s.dst, s.dst_col, s.dst_col + s.c_out):
                    zero.add(s.dst)   # a gradient read before anything wrote all of it
                if s.residual is not None:
                    rb, rc = s.residual
                    first_res[i] = write(rb, rc, rc + s.c_out)
                if i > 0:
                    first_dgrad[i] = write(s.src, s.src_col, s.src_col + s.c_in)
            if attempt == 0 and not zero:
                break
        # (the second attempt recomputes with the zeroed buffers forced to accumulate)
        self._plan = {"zero": sorted(zero), "res": first_res, "dgrad": first_dgrad}
        return self._plan

    def backward_layer(self, i, stream=None, parts=("wgrad", "residual", "dgrad")):
        s = self.layers[i]
        plan = self._first_touch()
        g = self.gbufs[s.dst][:, s.dst_col:s.dst_col + s.c_out]
        src = self.bufs[s.src][:, s.src_col:s.src_col + s.c_in]
        if "wgrad" in parts:
            spc.spc_conv_wgrad(self.maps[wgrad_map_key(s.map_key)], src, g, s.c_in, s.c_out, d_weight=self.dW[i],
                               stream=stream)
        if "residual" in parts and s.residual is not None:
            rb, rc = s.residual
            spc.spc_add_rows(self.gbufs[rb][:, rc:rc + s.c_out], g, stream=stream, accumulate=not plan["res"][i],
                             n_dev=self.level_n[s.level_out:s.level_out + 1])
        if "dgrad" in parts and i > 0:
            gsrc = self.gbufs[s.src][:, s.src_col:s.src_col + s.c_in]
            first = plan["dgrad"][i]
            spc.spc_conv_forward(self.maps[dgrad_map_key(s.map_key)], g, self.dgrad_weights[i], s.c_out, s.c_in,
                                 out=gsrc, residual=None if first else gsrc, ws=self.conv_ws, stream=stream)

    # ---------------------------------------------------------------------------------
    def algorithmic_flops(self) -> dict:
        """2 * nnz * C_in * C_out per layer (valid pairs only; OS sentinel rows not credited).
        [sync] -- exports every map once."""
        nnz, self.live_n = {}, {}
        for mk, km in self.maps.items():
            tr = spc.spc_kmap_export(km)
            nnz[mk] = int(tr.shape[0])
            # live sizes: every output row and every input row appears in >= 1 triple
            # (submanifold centre; strided / transposed K=3 s_l=2 parent offsets)
            self.live_n[mk] = (int(tr[:, 2].max()) + 1 if len(tr) else 0, int(tr[:, 1].max()) + 1 if len(tr) else 0)
        out = {}
        for s in self.layers:
            out[s.name] = 2.0 * nnz[s.map_key] * s.c_in_flops * s.c_out
        self.nnz = nnz
        return out

    def algorithmic_bytes(self) -> dict:
        """SURVEY 8(d) per layer: 2 N_in C_in + 2 N_out C_out (bf16 in/out) + 2 K^3 C_in C_out
        (weights) + 8 N_out C_out when the layer has a WS part (fp32 accumulator read + write).
        Call after algorithmic_flops()."""
        out = {}
        for s in self.layers:
            n_in, n_out = self.live_n[s.map_key]
            km = self.maps[s.map_key]
            b = 2 * n_in * s.c_in + 2 * n_out * s.c_out + 2 * s.map_key[0] ** 3 * s.c_in * s.c_out
            if km.c.n_lists > 0:
                b += 8 * n_out * s.c_out
            out[s.name] = float(b)
        return out


    def index_algorithmic_bytes(self) -> dict:
        """SURVEY 8(d) algorithmic bytes of the indexing phase of one pass (call after
        algorithmic_flops()): pack + sort 16 B in + 12 B out per voxel; each downsampled
        level 8 B read per input voxel + 8 B per unique output; each distinct kernel map
        8 N_in + 8 N_out (keys) + 4 N_out K_dense (OS table) + 8 per stored WS pair + 4 K^3."""
        n0 = int(self.level_n[0].item())
        ln = [int(v) for v in self.level_n.cpu().tolist()]
        out = {"pack_sort": 28.0 * n0, "downsample": float(sum(8 * n0 + 8 * m for m in ln[1:]))}
        maps = 0.0
        for mk, km in self.maps.items():
            n_in, n_out = self.live_n[mk]
            cnt = km.counts().cpu().numpy()
            pairs = int(cnt[spc.SPC_MAX_KVOL:spc.SPC_MAX_KVOL + km.n_lists].sum())
            maps += 8 * n_in + 8 * n_out + 4 * n_out * km.k_dense + 8 * pairs + 4 * km.k_vol
        out["kernel_maps"] = maps
        return out

    def nnz_per_out(self) -> dict:
        """Matches per output voxel of every distinct map (call after algorithmic_flops())."""
        return {mk: self.nnz[mk] / max(1, self.live_n[mk][1]) for mk in self.maps}


def pipeline_index_after(net) -> int:
    """The layer after which a pipelined step starts indexing the next scan: the first layer
    writing the deepest level, so the latency-bound indexing kernels overlap the small
    levels' latency-bound convolutions instead of the large levels' saturating ones (C2
    sweep of the start layer: 1.366 ms from the step start, 1.335 ms after the first
    deepest-level layer, 1.397 ms six layers later; scripts/pipeline_probe.py)."""
    deepest = max(s.level_out for s in net.layers)
    first = next(i for i, s in enumerate(net.layers) if s.level_out == deepest)
    # ... unless the deepest level is the network's tail (SECOND: 5 of 20 layers), where the
    # indexing would outlast the convolutions left (C3: 944 scans/s from the step start vs
    # 870 from its deepest level)
    return first if len(net.layers) - first >= 0.4 * len(net.layers) else -1


def capture_pipeline(nets, inputs, dev, stream, index_priority: int = 0, conv_priority: int = 0,
                     index_after_layer: int = -1):
    """Two CUDA graphs of a pipelined step: graph p runs nets[p].conv_stage (features of the
    scan nets[p] indexed in the previous step) on one stream and nets[1-p].index_stage on
    inputs[1-p] (the next scan) on another, forked from and joined into the capture stream."""
    s0 = torch.cuda.Stream(dev)
    s1 = torch.cuda.Stream(dev, priority=conv_priority)    # (< 0: higher scheduling priority)
    s2 = torch.cuda.Stream(dev, priority=index_priority)
    s0.wait_stream(stream)
    graphs = []
    for p in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s0):
            fork = torch.cuda.Event()
            fork.record(s0)
            s1.wait_event(fork)
            s2.wait_event(fork)
            mark = torch.cuda.Event() if index_after_layer >= 0 else None
            with torch.cuda.stream(s1):
                nets[p].conv_stage(s1, marks={index_after_layer: mark} if mark is not None else None)
            if mark is not None:   # start the indexing once the convolutions reach the small levels
                s2.wait_event(mark)
            with torch.cuda.stream(s2):
                c, f = inputs[1 - p]
                nets[1 - p].index_stage(c, f, s2)
            j1, j2 = torch.cuda.Event(), torch.cuda.Event()
            j1.record(s1)
            j2.record(s2)
            s0.wait_event(j1)
            s0.wait_event(j2)
        torch.cuda.synchronize()
        graphs.append(g)
    return graphs


def capture_pipeline3(nets, inputs, dev, stream, split: int):
    """Three scans in flight: graph p runs the layers [split, end) of nets[p] (scan i), the
    layers [0, split) of nets[p+1] (scan i+1) and the voxel indexing of nets[p+2] on
    inputs[p+2] (scan i+2), each on its own stream (three graphs, one per rotation)."""
    return capture_pipeline_n(nets, inputs, dev, stream, [split])


def capture_pipeline_n(nets, inputs, dev, stream, splits, index_after_layer: int = -1,
                       conv_max_ctas: int | None = None):
    """len(splits) + 2 scans in flight: a scan's convolutions are cut at `splits` into
    S = len(splits) + 1 segments; graph p runs segment S-1-k of nets[(p+k) % D] for k < S
    and the voxel indexing of nets[(p+S) % D] on inputs[(p+S) % D] (D = S + 1 instances),
    each on its own stream: every step finishes one scan and indexes one.
    conv_max_ctas: CTAs of the persistent feature kernels (SPC_OPT_CONV_MAX_CTAS) while
    capturing; None = SMs - 4, leaving a few SMs to the other streams' launches (C2 three in
    flight: 1.231 -> 1.202 ms at 142-146; 140: 1.207, 128: 1.209, uncapped 1.231); 0 = all."""
    if conv_max_ctas is None:
        conv_max_ctas = torch.cuda.get_device_properties(dev).multi_processor_count - 4
    caps = list(conv_max_ctas) if isinstance(conv_max_ctas, (list, tuple)) else [conv_max_ctas] * (len(splits) + 1)
    prev = spc.spc_get_option(spc.SPC_OPT_CONV_MAX_CTAS)
    try:
        return _capture_pipeline_n(nets, inputs, dev, stream, splits, index_after_layer, caps)
    finally:
        spc.spc_set_option(spc.SPC_OPT_CONV_MAX_CTAS, prev)


def _capture_pipeline_n(nets, inputs, dev, stream, splits, index_after_layer, caps):
    S = len(splits) + 1
    D = S + 1
    assert len(nets) == D and len(inputs) == D
    bounds = [0] + list(splits) + [None]
    s0 = torch.cuda.Stream(dev)
    ss = [torch.cuda.Stream(dev) for _ in range(D)]
    s0.wait_stream(stream)
    graphs = []
    for p in range(D):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s0):
            fork = torch.cuda.Event()
            fork.record(s0)
            for s in ss:
                s.wait_event(fork)
            mark = None
            for k in range(S):
                seg = S - 1 - k
                lo_, hi_ = bounds[seg], bounds[seg + 1]
                marks = None
                if index_after_layer >= lo_ and (hi_ is None or index_after_layer < hi_):
                    mark = torch.cuda.Event()   # the indexing starts once this layer is done
                    marks = {index_after_layer: mark}
                spc.spc_set_option(spc.SPC_OPT_CONV_MAX_CTAS, max(0, int(caps[seg])))   # (segment seg's cap)
                with torch.cuda.stream(ss[k]):
                    nets[(p + k) % D].conv_stage(ss[k], marks=marks, start=lo_, stop=hi_)
            if mark is not None:
                ss[S].wait_event(mark)
            with torch.cuda.stream(ss[S]):
                c, f = inputs[(p + S) % D]
                nets[(p + S) % D].index_stage(c, f, ss[S])
            for s in ss:
                j = torch.cuda.Event()
                j.record(s)
                s0.wait_event(j)
        torch.cuda.synchronize()
        graphs.append(g)
    return graphs


class SparseUNet(SparseNet):
    """MinkUNet-42 (configs C2, C4)."""

    def __init__(self, n0_cap: int, spec: spc.PackSpec, **kw):
        super().__init__(n0_cap, spec, net="minkunet42", **kw)
