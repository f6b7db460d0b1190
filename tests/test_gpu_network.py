"""Network-level GPU tests: full MinkUNet-42 / SECOND-K5 forward passes through the C ABI,
with layer-local parity (SURVEY §8(c) "Stacks"): a layer is recomputed by the oracle
from the GPU's own input to that layer, so bf16 error does not compound."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2511_20834_b200 as spc
from paper_2511_20834_b200.network import SparseNet, C_IN_PAD

pytestmark = pytest.mark.gpu


def _net(config, net_name, n_cut=None):
    coords = synth.make_scan(config, 0)
    if n_cut:
        coords = coords[:n_cut]
    spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
    net = SparseNet(coords.shape[0], spec, net=net_name)
    c_raw = 5 if net_name.startswith("second") else 4
    feats = torch.zeros(coords.shape[0], C_IN_PAD, dtype=torch.bfloat16, device="cuda")
    feats[:, :c_raw] = torch.from_numpy(synth.make_features(coords.shape[0], c_raw, seed=3)).cuda().bfloat16()
    out = net.forward(torch.from_numpy(coords).cuda(), feats)
    torch.cuda.synchronize()
    return net, coords, out


def _levels(coords, n_levels):
    c0 = oracle.sort_coords(coords)[0]
    return [c0] + [oracle.downsample(c0, 2 ** m) for m in range(1, n_levels)]


def _unpack_weight(net, i):
    """Recover W [K^3, C_in, C_out] from the seeded generator (same draw order as SparseNet)."""
    g = torch.Generator().manual_seed(20834)
    for j, s in enumerate(net.layers):
        kv = s.map_key[0] ** 3
        a = math.sqrt(3.0 / (min(kv, 10.0) * s.c_in_flops))
        w = (torch.rand(kv, s.c_in, s.c_out, generator=g) * 2 - 1) * a
        if s.c_in != s.c_in_flops:
            w[:, s.c_in_flops:, :] = 0
        if j == i:
            return w.bfloat16().float().numpy().astype(np.float64)
    raise IndexError(i)


def _layer_local(net, lv, i):
    s = net.layers[i]
    K, stride, ts, tr = s.map_key
    lf = int(round(math.log2(ts)))
    if stride == 1:
        inp = out = lv[lf]
    elif tr:
        inp, out = lv[lf + 1], lv[lf]
    else:
        inp, out = lv[lf], lv[lf + 1]
    src = net.bufs[s.src][: len(inp), s.src_col:s.src_col + s.c_in].float().cpu().numpy().astype(np.float64)
    net.conv(i)
    torch.cuda.synchronize()
    got = net.bufs[s.dst][: len(out), s.dst_col:s.dst_col + s.c_out].float().cpu().numpy().astype(np.float64)
    ref = oracle.conv(inp, out, K, ts, src, _unpack_weight(net, i), transposed=bool(tr))
    if s.residual is not None:
        rb, rc = s.residual
        ref = ref + net.bufs[rb][: len(out), rc:rc + s.c_out].float().cpu().numpy().astype(np.float64)
    # bf16-stored output: within one bf16 ulp of the fp64 reference (reading A18) + fp32 slack
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
    err = np.abs(got - ref) - ulp - 1e-5 * np.abs(ref).max()
    return float(err.max())


def test_minkunet42_forward_and_layer_local_parity():
    net, coords, out = _net(1, "minkunet42")
    assert torch.isfinite(out[: coords.shape[0]].float()).all()
    lv = _levels(coords, 5)
    names = [s.name for s in net.layers]
    for name in ("stem.conv1", "enc1.down", "enc2.rb1.proj", "enc2.rb1.conv2", "dec1.up", "dec4.rb1.conv1",
                 "dec4.rb2.conv2"):
        assert _layer_local(net, lv, names.index(name)) <= 0, name


def test_minkunet42_k2_forward_and_layer_local_parity():
    """TorchSparse's MinkUNet layer set: every K = 2 stride-2 down layer
    (offsets {0, s_p}^3) and K = 2 transposed up layer, plus neighbours."""
    net, coords, out = _net(1, "minkunet42_k2")
    assert torch.isfinite(out[: coords.shape[0]].float()).all()
    lv = _levels(coords, 5)
    names = [s.name for s in net.layers]
    for name in [f"enc{i}.down" for i in range(1, 5)] + [f"dec{j}.up" for j in range(1, 5)] + \
            ["enc1.rb1.conv1", "dec4.rb2.conv2"]:
        assert _layer_local(net, lv, names.index(name)) <= 0, name


def test_second_k5_backbone_forward_and_layer_local_parity():
    net, coords, out = _net(1, "secondk5")
    assert torch.isfinite(out[:1000].float()).all()
    lv = _levels(coords, 4)
    names = [s.name for s in net.layers]
    for name in ("stem", "s0.b0.conv1", "down1", "s1.b1.conv2", "s3.b0.conv1"):
        assert _layer_local(net, lv, names.index(name)) <= 0, name


def test_network_index_levels_match_oracle():
    net, coords, _ = _net(1, "minkunet42")
    lv = _levels(coords, 5)
    ln = net.level_n.cpu().tolist()
    assert ln == [len(x) for x in lv]


def _map_coords(lv, map_key):
    K, stride, ts, tr = map_key
    lf = int(round(math.log2(ts)))
    if stride == 1:
        return lv[lf], lv[lf], K, ts, False
    if tr:
        return lv[lf + 1], lv[lf], K, ts, True
    return lv[lf], lv[lf + 1], K, ts, False


@pytest.mark.parametrize("net_name", ["minkunet42", "secondk5"])
def test_training_backward_every_layer(net_name):
    """one forward + backward of the whole network (SparseNet(train=True):
    buffers versioned per write, dgrad on the forward / opposite-direction maps, wgrad,
    residual adds).  Every layer's weight gradient is recomputed by the oracle from the
    GPU's own forward input and output gradient (fp64, <= 2e-3 max|ref|); every activation
    gradient equals the sum the layer graph prescribes -- oracle dgrad of each reader plus
    the residual gradients -- within the bf16 storage of the running sum (1e-2 max|ref|)."""
    coords = synth.make_scan(1, 0)[:7000]
    spec = spc.spc_plan_pack(coords[:, 1:].min(0), coords[:, 1:].max(0), 1, 16, 16)
    net = SparseNet(coords.shape[0], spec, net=net_name, train=True)
    c_raw = 5 if net_name.startswith("second") else 4
    feats = torch.zeros(coords.shape[0], C_IN_PAD, dtype=torch.bfloat16, device="cuda")
    feats[:, :c_raw] = torch.from_numpy(synth.make_features(coords.shape[0], c_raw, seed=3)).cuda().bfloat16()
    net.forward(torch.from_numpy(coords).cuda(), feats)
    gout = torch.from_numpy(synth.make_features(coords.shape[0], net.bufs[net.out_name].shape[1], seed=4)).cuda()
    dW = net.backward(gout.bfloat16())
    torch.cuda.synchronize()
    lv = _levels(coords, net.n_levels)
    host = lambda t, n: t[:n].float().cpu().numpy().astype(np.float64)
    expect = {}   # (buffer) -> fp64 sum of every gradient contribution
    for i, s in enumerate(net.layers):
        inp, out, K, ts, tr = _map_coords(lv, s.map_key)
        g = host(net.gbufs[s.dst][:, s.dst_col:s.dst_col + s.c_out], len(out))
        src = host(net.bufs[s.src][:, s.src_col:s.src_col + s.c_in], len(inp))
        ref_w = oracle.conv_wgrad(inp, out, K, ts, src, g, transposed=tr)
        got_w = dW[i].cpu().numpy().astype(np.float64)
        m = np.abs(ref_w).max()
        assert np.abs(got_w - ref_w).max() <= 2e-3 * (m if m > 0 else 1), s.name
        if i > 0:
            W = _unpack_weight(net, i)
            d = oracle.conv_dgrad(inp, out, K, ts, g, W, transposed=tr)
            e = expect.setdefault(s.src, np.zeros((len(inp), net.gbufs[s.src].shape[1])))
            e[:, s.src_col:s.src_col + s.c_in] += d
        if s.residual is not None:
            rb, rc = s.residual
            e = expect.setdefault(rb, np.zeros((len(out), net.gbufs[rb].shape[1])))
            e[:, rc:rc + s.c_out] += g
    for name, ref in expect.items():
        got = host(net.gbufs[name], ref.shape[0])
        m = np.abs(ref).max()
        assert np.abs(got - ref).max() <= 1e-2 * m, name


def test_two_scans_in_flight_match_sequential():
    """capture_pipeline (the serving loop with two scans in flight: indexing of scan i+1
    on its own stream beside the convolutions of scan i, two network instances): with a
    deterministic configuration (all-OS maps, no split-K atomics) every output equals the
    sequential forward of the same scan bit for bit, for two different scans alternating."""
    from paper_2511_20834_b200.network import capture_pipeline
    scans = [synth.make_scan(1, 0)[:9000], synth.make_scan(1, 1)[:9000]]
    allc = np.concatenate(scans)
    spec = spc.spc_plan_pack(allc[:, 1:].min(0), allc[:, 1:].max(0), 1, 16, 16)
    spc.spc_set_option(spc.SPC_OPT_CONV_OS_SPLIT, 0)
    try:
        mk = lambda: SparseNet(9000, spec, t_override={k: spc.SPC_T_ALL_OS for k in
                                                       SparseNet(16, spec).map_keys})
        nets = [mk(), mk()]
        ins = []
        for s in scans:
            f = torch.zeros(s.shape[0], C_IN_PAD, dtype=torch.bfloat16, device="cuda")
            f[:, :4] = torch.from_numpy(synth.make_features(s.shape[0], 4, seed=s.shape[0])).cuda().bfloat16()
            ins.append((torch.from_numpy(s).cuda(), f))
        refs = []
        for c, f in ins:   # sequential reference, one scan at a time
            refs.append(nets[0].forward(c, f).clone())
        torch.cuda.synchronize()
        for q in range(2):
            nets[q].forward(*ins[q])
        nets[0].forward(*ins[0])   # scan 0 indexed in instance 0 (the pipeline's fill)
        torch.cuda.synchronize()
        graphs = capture_pipeline(nets, ins, torch.device("cuda"), torch.cuda.current_stream())
        nets[0].index_stage(*ins[0])
        for i in range(4):           # step i: features of scan i % 2 in nets[i % 2]
            graphs[i % 2].replay()
            torch.cuda.synchronize()
            assert torch.equal(nets[i % 2].bufs[nets[i % 2].out_name], refs[i % 2]), i
    finally:
        spc.spc_set_option(spc.SPC_OPT_CONV_OS_SPLIT, -1)


@pytest.mark.parametrize("caps", [None, 0, 140, [144, 136]])
def test_three_scans_in_flight_match_sequential(caps):
    """capture_pipeline3 (a scan's convolutions split at a layer: tail of scan i, head of
    scan i+1 and indexing of scan i+2 on three streams, three instances): with the
    deterministic configuration every output equals the sequential forward bit for bit,
    with the default CTA cap (SMs - 4), none, and per-segment caps."""
    from paper_2511_20834_b200.network import capture_pipeline_n
    scans = [synth.make_scan(1, s)[:9000] for s in range(3)]
    allc = np.concatenate(scans)
    spec = spc.spc_plan_pack(allc[:, 1:].min(0), allc[:, 1:].max(0), 1, 16, 16)
    spc.spc_set_option(spc.SPC_OPT_CONV_OS_SPLIT, 0)
    try:
        mk = lambda: SparseNet(9000, spec, t_override={k: spc.SPC_T_ALL_OS for k in
                                                       SparseNet(16, spec).map_keys})
        nets = [mk(), mk(), mk()]
        ins = []
        for s in scans:
            f = torch.zeros(s.shape[0], C_IN_PAD, dtype=torch.bfloat16, device="cuda")
            f[:, :4] = torch.from_numpy(synth.make_features(s.shape[0], 4, seed=s.shape[0])).cuda().bfloat16()
            ins.append((torch.from_numpy(s).cuda(), f))
        refs = [nets[0].forward(c, f).clone() for c, f in ins]
        torch.cuda.synchronize()
        for q in range(3):
            nets[q].forward(*ins[q])
        torch.cuda.synchronize()
        split = 22
        graphs = capture_pipeline_n(nets, ins, torch.device("cuda"), torch.cuda.current_stream(), [split],
                                    conv_max_ctas=caps)
        assert spc.spc_get_option(spc.SPC_OPT_CONV_MAX_CTAS) == 0   # restored after the capture
        # fill: scans 0 and 1 indexed, scan 0's first layers done
        nets[0].index_stage(*ins[0])
        nets[1].index_stage(*ins[1])
        nets[0].conv_stage(stop=split)
        for i in range(6):           # step i finishes scan i % 3 in nets[i % 3]
            graphs[i % 3].replay()
            torch.cuda.synchronize()
            assert torch.equal(nets[i % 3].bufs[nets[i % 3].out_name], refs[i % 3]), i
    finally:
        spc.spc_set_option(spc.SPC_OPT_CONV_OS_SPLIT, -1)
