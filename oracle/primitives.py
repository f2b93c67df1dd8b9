"""PETRA fp64 CPU oracle -- primitive layers and their hand-written VJPs.

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The CUDA path
(``paper_2406_02052_b200``) never imports it and shares no code with it.

Layout: NCHW, float64.  Every function is the plain definition written out;
library calls (``np.tensordot``) are used only as whole contraction steps.

Citations: PAPER.md line numbers (see /root/reference/PAPER.md at survey time);
readings of silent/ambiguous passages are numbered c1..c21 as in SURVEY.md §8(c)
and DESIGN.md "Readings".
"""
from __future__ import annotations

import numpy as np

BN_EPS = 1e-5        # reading c9 (paper silent; PyTorch default)
BN_MOMENTUM = 0.1    # reading c9

# The arithmetic of the bf16 tensor-core path (reading c22).  The paper
# fixes no precision (it trains in PyTorch's default fp32); north_star
# asks for bf16 tensor-core convolutions.  The oracle is exact fp64 by default.  Under
# ``bf16_convolutions()`` it follows ONE rule, stated here and in DESIGN.md, that
# names the rounding points of that path without asking the code under test:
#
#   R1  every convolution pass -- forward (and the recomputation), dgrad, wgrad --
#       rounds BOTH of its operands to bf16 (round-to-nearest-even of the fp32
#       value, :func:`bf16_round`) and then accumulates exactly;
#   R2  the forward result z is rounded to bf16 before BatchNorm reads it
#       (statistics, normalisation and the backward all see the rounded z);
#   R3  nothing else is rounded: streams, messages, BN, ReLU, the coupling add /
#       subtract, dgrad / wgrad results, the classifier and the optimizer stay exact.
#
# The ReLU masks are integers decided from floating point; under this rule both
# sides decide them on the same rounded operands (up to accumulation order).
#
# ``fp32_accumulation()`` (reading c25) changes the rounding, not the
# arithmetic: every convolution accumulates in fp32 (numpy's float32 contraction, a
# summation order of its own) and the tensors a device keeps in fp32 -- the stream
# halves after each coupling add / subtract, BN-ReLU activations, gradient sums -- are
# rounded to fp32 where they are produced (:func:`stored`).  It is not a model of any
# kernel; the tests use it to MEASURE how far an implementation of the same arithmetic
# that differs only in its rounding lands from the oracle -- through the ReLU masks
# such rounding moves.
_MODE = {"bf16": False, "acc32": False}


class bf16_convolutions:
    """Context manager: the oracle follows rules R1-R3 above while it is active."""

    def __enter__(self):
        self.prev = _MODE["bf16"]
        _MODE["bf16"] = True
        return self

    def __exit__(self, *exc):
        _MODE["bf16"] = self.prev


class fp32_accumulation:
    """Context manager: convolutions accumulate in fp32 while it is active (c25)."""

    def __enter__(self):
        self.prev = _MODE["acc32"]
        _MODE["acc32"] = True
        return self

    def __exit__(self, *exc):
        _MODE["acc32"] = self.prev


def _acc():
    return np.float32 if _MODE["acc32"] else np.float64


def stored(a):
    """A tensor the device keeps in fp32: rounded to fp32 under fp32_accumulation()."""
    return np.asarray(a, np.float32).astype(np.float64) if _MODE["acc32"] else a


def bf16_round(a):
    """Round to bfloat16 (8 significand bits, 8 exponent bits; IEEE round to nearest,
    ties to even), through fp32 (device operands are fp32 values), returned as fp64.

    Written from the definition: a finite fp32 value v with binary exponent
    e = floor(log2|v|) (clamped to -126, the subnormal range) lies on the bf16 grid
    of spacing ulp = 2^(e-7); v/ulp is rounded half-to-even; results of magnitude
    >= 2^128 overflow to inf.  NaN and inf pass through."""
    v = np.asarray(a, np.float32).astype(np.float64)
    out = v.copy()
    fin = np.isfinite(v) & (v != 0)
    e = np.frexp(v[fin])[1] - 1.0            # v = m * 2^e, 1 <= |m| < 2 (exact)
    e = np.maximum(e, -126.0)
    ulp = np.exp2(e - 7.0)
    r = np.round(v[fin] / ulp) * ulp        # numpy rounds half to even
    r[np.abs(r) >= 2.0 ** 128] = np.inf * np.sign(r[np.abs(r) >= 2.0 ** 128])
    out[fin] = r
    return out


def _op(a):
    """A convolution operand / forward result under the active precision (R1, R2)."""
    return bf16_round(a) if _MODE["bf16"] else a


# --------------------------------------------------------------------------- conv
def conv_out_size(n: int, k: int, stride: int, pad: int) -> int:
    return (n + 2 * pad - k) // stride + 1


def _taps(xp, k, stride, Ho, Wo):
    """Yield (kh, kw, view) with view[b,c,i,j] = xp[b,c,i*s+kh,j*s+kw]."""
    for kh in range(k):
        for kw in range(k):
            yield kh, kw, xp[:, :, kh:kh + stride * (Ho - 1) + 1:stride,
                             kw:kw + stride * (Wo - 1) + 1:stride]


def conv2d(x, w, stride=1, pad=0):
    """2-D cross-correlation without bias (the convolutions of F, G, the stem and
    the projections; "3x3 convolutions"):

        out[b,o,i,j] = sum_{c,kh,kw} w[o,c,kh,kw] * xpad[b,c,i*s+kh,j*s+kw]

    x: [B,C,H,W], w: [O,C,k,k]  ->  [B,O,Ho,Wo],  Ho = floor((H+2p-k)/s)+1.
    """
    B, C, H, W = x.shape
    O, C2, k, k2 = w.shape
    if C != C2 or k != k2:
        raise ValueError(f"conv2d shape mismatch x{x.shape} w{w.shape}")
    Ho, Wo = conv_out_size(H, k, stride, pad), conv_out_size(W, k, stride, pad)
    x, w = _op(x), _op(w)                                  # R1
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    dt = _acc()
    xp, w = xp.astype(dt, copy=False), w.astype(dt, copy=False)
    out = np.zeros((B, O, Ho, Wo), dt)
    for kh, kw, view in _taps(xp, k, stride, Ho, Wo):
        # sum over c of view[b,c,i,j] * w[o,c,kh,kw]  -> [B,Ho,Wo,O]
        out += np.tensordot(view, w[:, :, kh, kw], axes=([1], [1])).transpose(0, 3, 1, 2)
    out = out.astype(np.float64, copy=False)
    return _op(out)                                        # R2


def conv2d_vjp(x, w, stride, pad, dout, need_dx=True):
    """VJP of :func:`conv2d` (Eqs. 2-3, lines 74 and 79, applied to one conv):

        dW[o,c,kh,kw] = sum_{b,i,j} dout[b,o,i,j] * xpad[b,c,i*s+kh,j*s+kw]
        dxpad[b,c,i*s+kh,j*s+kw] += sum_o dout[b,o,i,j] * w[o,c,kh,kw]
    """
    B, C, H, W = x.shape
    O, _, k, _ = w.shape
    Ho, Wo = dout.shape[2], dout.shape[3]
    xw, dw_out = _op(x), _op(dout)                         # R1 (wgrad operands)
    dd_out, wd = _op(dout), _op(w)                         # R1 (dgrad operands)
    xp = np.pad(xw, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    dt = _acc()
    xp, dw_out = xp.astype(dt, copy=False), dw_out.astype(dt, copy=False)
    dd_out, wd = dd_out.astype(dt, copy=False), wd.astype(dt, copy=False)
    dxp = np.zeros(xp.shape, dt) if need_dx else None
    dw = np.zeros(w.shape, dt)
    for kh, kw, view in _taps(xp, k, stride, Ho, Wo):
        dw[:, :, kh, kw] = np.tensordot(dw_out, view, axes=([0, 2, 3], [0, 2, 3]))
        if need_dx:
            contrib = np.tensordot(dd_out, wd[:, :, kh, kw], axes=([1], [0]))  # [B,Ho,Wo,C]
            dxp[:, :, kh:kh + stride * (Ho - 1) + 1:stride,
                kw:kw + stride * (Wo - 1) + 1:stride] += contrib.transpose(0, 3, 1, 2)
    dx = dxp[:, :, pad:pad + H, pad:pad + W].astype(np.float64) if need_dx else None
    return dx, dw.astype(np.float64, copy=False)


# --------------------------------------------------------------------------- batch norm
def bn_train_forward(z, gamma, beta, eps=BN_EPS):
    """BatchNorm in training mode with batch statistics over (B,H,W) (reading c9:
    biased variance for normalisation).  Returns (out, cache)."""
    axes = (0, 2, 3)
    mu = z.mean(axis=axes)
    var = ((z - mu[None, :, None, None]) ** 2).mean(axis=axes)
    invstd = 1.0 / np.sqrt(var + eps)
    xhat = (z - mu[None, :, None, None]) * invstd[None, :, None, None]
    out = gamma[None, :, None, None] * xhat + beta[None, :, None, None]
    return out, {"xhat": xhat, "invstd": invstd, "mu": mu, "var": var, "n": z.size // z.shape[1]}


def bn_running_update(rmean, rvar, cache, momentum=BN_MOMENTUM):
    """EMA of the running statistics (reading c9: unbiased variance, momentum 0.1).
    Called ONLY when activations are recomputed in the backward (PAPER.md:259:
    "updated when recomputing the activations during the backward pass ... not
    updated during the forward pass"), or in the last stage's single forward (c10)."""
    n = cache["n"]
    rmean *= (1.0 - momentum)
    rmean += momentum * cache["mu"]
    rvar *= (1.0 - momentum)
    rvar += momentum * cache["var"] * n / max(n - 1, 1)


def bn_train_vjp(cache, gamma, dout):
    """Closed-form VJP of training-mode BN (running stats are constants):
        dbeta = sum g,  dgamma = sum g*xhat,
        dz = gamma*invstd*(g - mean(g) - xhat*mean(g*xhat)),   g = dout."""
    axes = (0, 2, 3)
    xhat, invstd = cache["xhat"], cache["invstd"]
    dbeta = dout.sum(axis=axes)
    dgamma = (dout * xhat).sum(axis=axes)
    n = cache["n"]
    dz = (gamma * invstd)[None, :, None, None] * (
        dout - (dbeta / n)[None, :, None, None] - xhat * (dgamma / n)[None, :, None, None])
    return dz, dgamma, dbeta


# --------------------------------------------------------------------------- relu / pool
# ReLU-mask instrumentation for the flip-floor derivation (reading c25).
# ``MASKS["record"]``: a list that receives every mask decided; ``MASKS["replay"]``: a
# list of masks consumed in order instead of deciding them (the same code path run
# twice calls relu in the same order); ``MASKS["band"]``: tau -- every decision whose
# pre-activation lies within tau * rms(a) of zero is taken the other way.  All None
# (the default): plain ReLU.
MASKS = {"record": None, "replay": None, "band": None}


def relu(a):
    """ReLU with mask a > 0 (reading c19: derivative 0 at 0)."""
    mask = a > 0
    if MASKS["band"] is not None:
        near = np.abs(a) <= MASKS["band"] * np.sqrt(np.mean(a * a))
        mask = mask ^ near
    if MASKS["replay"] is not None:
        m = MASKS["replay"].pop(0)
        if m.shape != mask.shape:
            raise ValueError(f"mask replay out of order: {m.shape} vs {mask.shape}")
        mask = m
    if MASKS["record"] is not None:
        MASKS["record"].append(mask.copy())
    return np.where(mask, a, 0.0), mask


def maxpool3x3s2(x):
    """Max-pool 3x3, stride 2, pad 1 (ImageNet stem, PAPER.md:259 contrast with CIFAR).
    Ties: first index in row-major window order.  Returns (out, argmax)."""
    B, C, H, W = x.shape
    Ho, Wo = conv_out_size(H, 3, 2, 1), conv_out_size(W, 3, 2, 1)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=-np.inf)
    best = np.full((B, C, Ho, Wo), -np.inf)
    arg = np.zeros((B, C, Ho, Wo), dtype=np.int64)
    for kh in range(3):
        for kw in range(3):
            v = xp[:, :, kh:kh + 2 * (Ho - 1) + 1:2, kw:kw + 2 * (Wo - 1) + 1:2]
            upd = v > best  # strict: keeps the first maximum
            best = np.where(upd, v, best)
            arg = np.where(upd, kh * 3 + kw, arg)
    return best, arg


def maxpool3x3s2_vjp(x_shape, arg, dout):
    B, C, H, W = x_shape
    Ho, Wo = dout.shape[2:]
    dxp = np.zeros((B, C, H + 2, W + 2))
    for kh in range(3):
        for kw in range(3):
            sel = (arg == kh * 3 + kw)
            dxp[:, :, kh:kh + 2 * (Ho - 1) + 1:2, kw:kw + 2 * (Wo - 1) + 1:2] += np.where(sel, dout, 0.0)
    return dxp[:, :, 1:1 + H, 1:1 + W].copy()


# --------------------------------------------------------------------------- head / loss
def linear(x, w, b):
    """y = x w^T + b (the classifier, "L <- F_J(x_{J-1}, theta_J)")."""
    return x @ w.T + b


def softmax_cross_entropy(logits, labels):
    """Batch-mean softmax cross-entropy (reading c18) and its gradient
    dlogits = (softmax - onehot) / B."""
    B = logits.shape[0]
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    s = e.sum(axis=1, keepdims=True)
    logp = logits - m - np.log(s)
    loss = -logp[np.arange(B), labels].mean()
    p = e / s
    p[np.arange(B), labels] -= 1.0
    return float(loss), p / B
