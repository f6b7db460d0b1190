"""Pins for the oracle's NEXT-4 functions (training path and fused epilogue): the gradients
of Eq. (2) against torch autograd of conv3d / conv_transpose3d in float64 on
dense grids read at the sparse sites, and the BN / residual / ReLU epilogue against
torch.nn.functional.batch_norm (eval) + relu.  CPU only (-m "not gpu")."""
import numpy as np
import pytest
import torch

import oracle
import synth


def _dense_w(W, ks):
    # weight[co, ci, ex, ey, ez] = W[k(e), ci, co], k lexicographic (ex, ey, ez), ez fastest
    kv, ci, co = W.shape
    return torch.from_numpy(W.reshape(*ks, ci, co)).permute(4, 3, 0, 1, 2).contiguous()


def _w_back(g, ks):
    # inverse of _dense_w for a [co, ci, kx, ky, kz] gradient
    co, ci = g.shape[0], g.shape[1]
    return g.permute(2, 3, 4, 1, 0).reshape(ks[0] * ks[1] * ks[2], ci, co).numpy()


def _scatter(coords, F, size, div=1):
    g = torch.zeros((1, F.shape[1]) + size, dtype=torch.float64)
    for r, (_, x, y, z) in enumerate(coords.tolist()):
        g[0, :, x // div, y // div, z // div] = torch.from_numpy(F[r])
    return g


def _autograd(fine, coarse_or_out, F, G, W, ks, kind):
    """loss = sum_i <y(out_i), G_i> through a dense float64 torch convolution; returns
    (dF_in at the input sites, dW in [kv, c_in, c_out])."""
    n = 8
    pad = tuple((k - 1) // 2 if k % 2 else 0 for k in ks)
    w = _dense_w(W, ks).requires_grad_(True)
    if kind == "subm":
        x = _scatter(fine, F, (n, n, n)).requires_grad_(True)
        y = torch.nn.functional.conv3d(x, w, padding=pad)
        out_idx = [(a, b, c) for _, a, b, c in coarse_or_out.tolist()]
        in_idx = [(a, b, c) for _, a, b, c in fine.tolist()]
    elif kind == "down":
        x = _scatter(fine, F, (n, n, n)).requires_grad_(True)
        y = torch.nn.functional.conv3d(x, w, stride=2, padding=pad)
        out_idx = [(a // 2, b // 2, c // 2) for _, a, b, c in coarse_or_out.tolist()]
        in_idx = [(a, b, c) for _, a, b, c in fine.tolist()]
    else:   # "up": coarse inputs (F rows) -> fine outputs, same weight index as "down"
        x = _scatter(fine, F, (n // 2,) * 3, div=2).requires_grad_(True)
        wt = w.permute(1, 0, 2, 3, 4)   # conv_transpose3d weight [c_in, c_out, ...]
        op = tuple(1 if k % 2 else 0 for k in ks)
        y = torch.nn.functional.conv_transpose3d(x, wt, stride=2, padding=pad, output_padding=op)
        out_idx = [(a, b, c) for _, a, b, c in coarse_or_out.tolist()]
        in_idx = [(a // 2, b // 2, c // 2) for _, a, b, c in fine.tolist()]
    loss = sum((y[0, :, a, b, c] * torch.from_numpy(G[r])).sum() for r, (a, b, c) in enumerate(out_idx))
    loss.backward()
    dF = np.stack([x.grad[0, :, a, b, c].numpy() for a, b, c in in_idx])
    return dF, _w_back(w.grad, ks)


def _cloud(seed, n=140):
    return oracle.sort_coords(synth.random_cloud(n, 8, seed=seed, signed=False))[0]


@pytest.mark.parametrize("ks", [(3, 3, 3), (3, 1, 1), (1, 1, 1)])
def test_grads_submanifold_vs_autograd(ks):
    rng = np.random.default_rng(sum(ks))
    c = _cloud(3 + ks[1])
    F = rng.uniform(-1, 1, (len(c), 5))
    G = rng.uniform(-1, 1, (len(c), 6))
    W = rng.uniform(-1, 1, (ks[0] * ks[1] * ks[2], 5, 6))
    K = ks[0] if ks[0] == ks[1] == ks[2] else ks
    dF, dW = _autograd(c, c, F, G, W, ks, "subm")
    np.testing.assert_allclose(oracle.conv_dgrad(c, c, K, 1, G, W), dF, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_wgrad(c, c, K, 1, F, G), dW, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("ks", [(3, 3, 3), (2, 2, 2)])
def test_grads_strided_and_transposed_vs_autograd(ks):
    rng = np.random.default_rng(ks[0] + 10)
    fine = _cloud(ks[0] + 20, 180)
    coarse = oracle.downsample(fine, 2)
    K = ks[0] if ks[0] % 2 else ks
    # down: fine in -> coarse out
    F = rng.uniform(-1, 1, (len(fine), 4))
    G = rng.uniform(-1, 1, (len(coarse), 3))
    W = rng.uniform(-1, 1, (ks[0] ** 3, 4, 3))
    dF, dW = _autograd(fine, coarse, F, G, W, ks, "down")
    np.testing.assert_allclose(oracle.conv_dgrad(fine, coarse, K, 1, G, W), dF, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_wgrad(fine, coarse, K, 1, F, G), dW, rtol=1e-12, atol=1e-12)
    # up (transposed): coarse in -> fine out
    Fc = rng.uniform(-1, 1, (len(coarse), 3))
    Gf = rng.uniform(-1, 1, (len(fine), 4))
    Wt = rng.uniform(-1, 1, (ks[0] ** 3, 3, 4))
    dFc, dWt = _autograd(coarse, fine, Fc, Gf, Wt, ks, "up")
    np.testing.assert_allclose(oracle.conv_dgrad(coarse, fine, K, 1, Gf, Wt, transposed=True), dFc,
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_wgrad(coarse, fine, K, 1, Fc, Gf, transposed=True), dWt,
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kind", ["subm", "down", "up"])
def test_dgrad_rows_gather_equals_scatter(kind):
    """The gather form (hash on the output set) and the scatter form (hash on the input
    set) share only the definition."""
    rng = np.random.default_rng(5)
    fine = _cloud(31, 300)
    coarse = oracle.downsample(fine, 2)
    a, b, tr = {"subm": (fine, fine, False), "down": (fine, coarse, False), "up": (coarse, fine, True)}[kind]
    G = rng.uniform(-1, 1, (len(b), 7))
    W = rng.uniform(-1, 1, (27, 4, 7))
    full = oracle.conv_dgrad(a, b, 3, 1, G, W, transposed=tr)
    rows = np.array([0, 3, len(a) // 2, len(a) - 1])
    np.testing.assert_allclose(oracle.conv_dgrad_rows(a, b, rows, 3, 1, G, W, transposed=tr), full[rows],
                               rtol=1e-13, atol=1e-13)


def test_grad_identities():
    """dgrad is the adjoint of Eq. (2): <conv(F), G> = <F, dgrad(G)> = <W, wgrad(F, G)>."""
    rng = np.random.default_rng(9)
    c = _cloud(41, 250)
    F = rng.uniform(-1, 1, (len(c), 6))
    G = rng.uniform(-1, 1, (len(c), 5))
    W = rng.uniform(-1, 1, (27, 6, 5))
    y = oracle.conv(c, c, 3, 1, F, W)
    lhs = float((y * G).sum())
    assert abs(lhs - float((F * oracle.conv_dgrad(c, c, 3, 1, G, W)).sum())) < 1e-9 * max(1, abs(lhs))
    assert abs(lhs - float((W * oracle.conv_wgrad(c, c, 3, 1, F, G)).sum())) < 1e-9 * max(1, abs(lhs))
    # K = 1: dgrad = G W^T, wgrad = F^T G
    W1 = rng.uniform(-1, 1, (1, 6, 5))
    np.testing.assert_allclose(oracle.conv_dgrad(c, c, 1, 1, G, W1), G @ W1[0].T, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(oracle.conv_wgrad(c, c, 1, 1, F, G)[0], F.T @ G, rtol=1e-12, atol=1e-12)


def test_bn_relu_vs_torch():
    rng = np.random.default_rng(3)
    x = rng.normal(0, 2, (200, 24))
    res = rng.normal(0, 1, (200, 24))
    gamma, beta = rng.uniform(0.5, 2, 24), rng.normal(0, 1, 24)
    mean, var = rng.normal(0, 1, 24), rng.uniform(0.1, 3, 24)
    t = lambda a: torch.from_numpy(a)
    bn = torch.nn.functional.batch_norm(t(x), t(mean), t(var), t(gamma), t(beta), training=False, eps=1e-3)
    np.testing.assert_allclose(oracle.bn_relu(x, gamma, beta, mean, var, 1e-3, relu=False), bn.numpy(),
                               rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(oracle.bn_relu(x, gamma, beta, mean, var, 1e-3, residual=res),
                               torch.relu(bn + t(res)).numpy(), rtol=1e-13, atol=1e-13)
    np.testing.assert_array_equal(oracle.bn_relu(x), np.maximum(x, 0))
