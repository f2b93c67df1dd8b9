"""Pins of the oracle primitives against things other than the oracle itself:
worked examples (tests/golden), brute-force loops, torch.nn.functional in fp64
(an independent library), central finite differences (h=1e-5,
rel 1e-4)."""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as TF

from oracle import primitives as P
import synth


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def t64(a):
    return torch.tensor(np.asarray(a), dtype=torch.float64, requires_grad=True)


# --------------------------------------------------------------------- conv
def test_conv_worked_example(golden):
    g = golden("conv_ones.json")
    out = P.conv2d(np.ones(g["x_shape"]), np.ones(g["w_shape"]), g["stride"], g["pad"])
    assert out.tolist() == g["out"]


def brute_conv(x, w, s, p):
    B, C, H, W = x.shape
    O, _, k, _ = w.shape
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    out = np.zeros((B, O, Ho, Wo))
    for b, o, i, j in itertools.product(range(B), range(O), range(Ho), range(Wo)):
        acc = 0.0
        for c, kh, kw in itertools.product(range(C), range(k), range(k)):
            hi, wi = i * s + kh - p, j * s + kw - p
            if 0 <= hi < H and 0 <= wi < W:
                acc += w[o, c, kh, kw] * x[b, c, hi, wi]
        out[b, o, i, j] = acc
    return out


@pytest.mark.parametrize("k,s,H", [(3, 1, 5), (3, 2, 6), (1, 1, 4), (1, 2, 5), (7, 2, 9)])
def test_conv_brute_force(k, s, H):
    x = synth.normal((2, 3, H, H + 1), 0, k, s)
    w = synth.normal((4, 3, k, k), 1, k, s)
    p = (k - 1) // 2
    np.testing.assert_allclose(P.conv2d(x, w, s, p), brute_conv(x, w, s, p), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("k,s", [(3, 1), (3, 2), (1, 2), (7, 2)])
def test_conv_vs_torch_and_vjp(k, s):
    p = (k - 1) // 2
    x = synth.normal((2, 5, 9, 8), 3, k, s)
    w = synth.normal((6, 5, k, k), 4, k, s)
    dout_shape = P.conv2d(x, w, s, p).shape
    dout = synth.normal(dout_shape, 5, k, s)
    xt, wt = t64(x), t64(w)
    yt = TF.conv2d(xt, wt, stride=s, padding=p)
    assert rel(P.conv2d(x, w, s, p), yt.detach().numpy()) < 1e-13
    yt.backward(torch.tensor(dout))
    dx, dw = P.conv2d_vjp(x, w, s, p, dout)
    assert rel(dx, xt.grad.numpy()) < 1e-13
    assert rel(dw, wt.grad.numpy()) < 1e-13


def fd_check(f, x, direction, h=1e-5):
    """Central difference of scalar f along ``direction``."""
    return (f(x + h * direction) - f(x - h * direction)) / (2 * h)


def test_conv_vjp_finite_difference():
    x = synth.normal((1, 2, 5, 5), 6)
    w = synth.normal((3, 2, 3, 3), 7)
    dout = synth.normal((1, 3, 3, 3), 8)
    dx, dw = P.conv2d_vjp(x, w, 2, 1, dout)
    for trial in range(3):
        u = synth.normal(x.shape, 9, trial)
        fd = fd_check(lambda xx: np.sum(P.conv2d(xx, w, 2, 1) * dout), x, u)
        assert abs(fd - np.sum(dx * u)) <= 1e-4 * abs(fd) + 1e-10
        v = synth.normal(w.shape, 10, trial)
        fd = fd_check(lambda ww: np.sum(P.conv2d(x, ww, 2, 1) * dout), w, v)
        assert abs(fd - np.sum(dw * v)) <= 1e-4 * abs(fd) + 1e-10


# --------------------------------------------------------------------- batch norm
def test_bn_normalised_input_is_identity():
    """per-channel mean 0 / var 1 input, gamma=1, beta=0 -> output ~= x."""
    z = synth.normal((8, 3, 4, 4), 11)
    z = (z - z.mean(axis=(0, 2, 3), keepdims=True)) / z.std(axis=(0, 2, 3), keepdims=True)
    out, _ = P.bn_train_forward(z, np.ones(3), np.zeros(3))
    # closed form: exactly z / sqrt(1 + eps) (biased var of normalised z is 1)
    np.testing.assert_allclose(out, z / np.sqrt(1 + 1e-5), rtol=1e-13, atol=1e-14)
    assert np.max(np.abs(out - z)) < 1e-5 * np.max(np.abs(z))


def test_bn_vs_torch_forward_vjp_running_stats():
    z = synth.normal((4, 5, 3, 3), 12) * 3 + 1
    gamma = synth.normal((5,), 13) + 1
    beta = synth.normal((5,), 14)
    dout = synth.normal(z.shape, 15)
    zt, gt, bt = t64(z), t64(gamma), t64(beta)
    rm_t, rv_t = torch.zeros(5, dtype=torch.float64), torch.ones(5, dtype=torch.float64)
    yt = TF.batch_norm(zt, rm_t, rv_t, gt, bt, training=True, momentum=0.1, eps=1e-5)
    yt.backward(torch.tensor(dout))
    out, cache = P.bn_train_forward(z, gamma, beta)
    assert rel(out, yt.detach().numpy()) < 1e-13
    dz, dg, db = P.bn_train_vjp(cache, gamma, dout)
    assert rel(dz, zt.grad.numpy()) < 1e-12
    assert rel(dg, gt.grad.numpy()) < 1e-13
    assert rel(db, bt.grad.numpy()) < 1e-13
    rm, rv = np.zeros(5), np.ones(5)
    P.bn_running_update(rm, rv, cache)
    assert rel(rm, rm_t.numpy()) < 1e-14
    assert rel(rv, rv_t.numpy()) < 1e-14


def test_bn_running_stats_geometric_convergence():
    """EMA on a constant batch converges geometrically to the batch mean."""
    z = synth.normal((16, 2, 2, 2), 16) + 3.0
    _, cache = P.bn_train_forward(z, np.ones(2), np.zeros(2))
    rm, rv = np.zeros(2), np.ones(2)
    gaps = []
    for _ in range(5):
        P.bn_running_update(rm, rv, cache)
        gaps.append(np.abs(rm - cache["mu"]))
    for a, b in zip(gaps, gaps[1:]):
        np.testing.assert_allclose(b, 0.9 * a, rtol=1e-12)


def test_bn_vjp_finite_difference():
    z = synth.normal((3, 2, 2, 3), 17)
    gamma, beta = np.array([1.3, 0.7]), np.array([0.1, -0.2])
    dout = synth.normal(z.shape, 18)
    _, cache = P.bn_train_forward(z, gamma, beta)
    dz, _, _ = P.bn_train_vjp(cache, gamma, dout)
    u = synth.normal(z.shape, 19)
    fd = fd_check(lambda zz: np.sum(P.bn_train_forward(zz, gamma, beta)[0] * dout), z, u)
    assert abs(fd - np.sum(dz * u)) <= 1e-4 * abs(fd) + 1e-9


# --------------------------------------------------------------------- relu / maxpool
def test_relu_subgradient():
    """relu x=[-1,2], delta=[5,5] -> [0,5]; reading c19: 0 at 0."""
    y, mask = P.relu(np.array([-1.0, 2.0, 0.0]))
    assert y.tolist() == [0.0, 2.0, 0.0]
    assert (np.array([5.0, 5.0, 5.0]) * mask).tolist() == [0.0, 5.0, 0.0]


def test_maxpool_vs_torch():
    x = synth.normal((2, 3, 9, 8), 20)
    xt = t64(x)
    yt = TF.max_pool2d(xt, 3, 2, 1)
    out, arg = P.maxpool3x3s2(x)
    assert rel(out, yt.detach().numpy()) == 0.0
    dout = synth.normal(out.shape, 21)
    yt.backward(torch.tensor(dout))
    assert rel(P.maxpool3x3s2_vjp(x.shape, arg, dout), xt.grad.numpy()) < 1e-15


def test_maxpool_first_index_ties():
    """ties go to the first index in row-major window order."""
    x = np.zeros((1, 1, 3, 3))
    out, arg = P.maxpool3x3s2(x)
    # output (0,0) window covers padded rows/cols -1..1; first in-bounds max is (0,0) = tap (1,1)
    assert arg[0, 0, 0, 0] == 4
    d = P.maxpool3x3s2_vjp(x.shape, arg, np.ones(out.shape))
    assert d.sum() == out.size and d[0, 0, 0, 0] == 1.0


# --------------------------------------------------------------------- loss
def test_ce_uniform_is_log_c():
    loss, d = P.softmax_cross_entropy(np.zeros((4, 10)), np.array([0, 3, 9, 2]))
    assert abs(loss - np.log(10)) < 1e-15
    np.testing.assert_allclose(d.sum(axis=1), 0.0, atol=1e-16)


def test_ce_vs_torch():
    logits = synth.normal((6, 7), 22) * 3
    lab = synth.labels(6, 7, 23)
    lt = t64(logits)
    lt_loss = TF.cross_entropy(lt, torch.tensor(lab))
    lt_loss.backward()
    loss, d = P.softmax_cross_entropy(logits, lab)
    assert abs(loss - lt_loss.item()) < 1e-14
    assert rel(d, lt.grad.numpy()) < 1e-14
    np.testing.assert_allclose(d.sum(axis=1), 0.0, atol=1e-15)
