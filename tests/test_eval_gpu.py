"""Evaluation forward (petra_stage_eval / petra_stage_eval_tail; the running
statistics of BN "are then used during model evaluation").

Reference: the unit written out with the oracle's primitives, BN normalising by the
RUNNING mean / variance (x_hat = (z - rm) / sqrt(rv + eps)) instead of the batch
statistics; the classifier's first-index argmax against the labels and the batch-mean
cross-entropy.  The evaluation must leave every parameter, optimizer slot and running
statistic bitwise unchanged."""
import numpy as np
import pytest

import synth
from oracle import primitives as OP
from oracle.units import Branch, ConvBN, RevUnit, TailUnit
from tests.gpu_harness import nchw, nhwc, oracle_to_product_units, pack_params, rand_params, rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2406_02052_b200 import Stage  # noqa: E402
from paper_2406_02052_b200 import _lib as L  # noqa: E402
from paper_2406_02052_b200 import models as PM  # noqa: E402


def _units(tail):
    u = [RevUnit(0, Branch([ConvBN(64, 64, 3, 1)])), RevUnit(1, Branch([ConvBN(64, 64, 3, 1)]))]
    if tail:
        u.append(TailUnit(128, 10))
    rand_params(u, 7)
    for i, x in enumerate(u[:2]):  # running statistics away from (0, 1)
        L0 = x.phi.layers[0]
        L0.rmean[...] = 0.3 * synth.normal(L0.rmean.shape, 7, 200, i)
        L0.rvar[...] = 0.5 + np.abs(synth.normal(L0.rvar.shape, 7, 201, i))
    if tail:
        u[2].b[...] = 0.1 * synth.normal(u[2].b.shape, 7, 202, 0)
    return u


def _ref_forward(units, xs):
    xs = [a.astype(np.float64) for a in xs]
    for u in units:
        if not isinstance(u, RevUnit):
            continue
        c = u.phi.layers[0]
        z = OP.conv2d(xs[u.src], c.w, c.stride, c.pad)
        sh = (1, -1, 1, 1)
        y = c.gamma.reshape(sh) * (z - c.rmean.reshape(sh)) / np.sqrt(c.rvar.reshape(sh) + OP.BN_EPS) + \
            c.beta.reshape(sh)
        xs[u.dst] = xs[u.dst] + np.maximum(y, 0.0)
    return xs


def _stage(units, B, precision):
    spec = PM.StageSpec(oracle_to_product_units(units), B, (16, 16, 64), precision)
    st = Stage(spec, 0)
    th, bf = pack_params(units)
    st.set_params(th, np.zeros_like(th), bf)
    return st


@pytest.mark.parametrize("precision", [L.FP32, L.BF16_TC], ids=["fp32", "bf16"])
def test_stage_eval_running_statistics(precision):
    torch.cuda.set_device(0)
    B = 4
    units = _units(False)
    st = _stage(units, B, precision)
    xs = [synth.images((B, 64, 16, 16), 3, h) for h in range(2)]
    before = st.get_params()
    d = [torch.tensor(nhwc(x), dtype=torch.float32, device="cuda") for x in xs]
    o = [torch.empty_like(d[0]) for _ in range(2)]
    st.eval(d[0], d[1], o[0], o[1])
    torch.cuda.synchronize()
    ref = _ref_forward(units, xs)
    tol = 1e-4 if precision == L.FP32 else 2e-2
    for h in range(2):
        assert rel(nchw(o[h].cpu().numpy()), ref[h]) < tol, h
    after = st.get_params()
    for a, b in zip(before, after):
        assert np.array_equal(a, b)
    st.close()


@pytest.mark.parametrize("precision", [L.FP32, L.BF16_TC], ids=["fp32", "bf16"])
def test_stage_eval_tail_accuracy_and_loss(precision):
    torch.cuda.set_device(0)
    B = 16
    units = _units(True)
    st = _stage(units, B, precision)
    xs = [synth.images((B, 64, 16, 16), 4, h) for h in range(2)]
    labels = synth.labels(B, 10, 4, 0)
    before = st.get_params()
    d = [torch.tensor(nhwc(x), dtype=torch.float32, device="cuda") for x in xs]
    lab = torch.tensor(labels, dtype=torch.int32, device="cuda")
    correct = torch.zeros(1, dtype=torch.int32, device="cuda")
    loss = torch.zeros(1, device="cuda")
    st.eval_tail(d[0], d[1], lab, correct, loss)
    st.eval_tail(d[0], d[1], lab, correct, loss)  # accumulates
    torch.cuda.synchronize()
    feats = _ref_forward(units, xs)
    feat = np.concatenate([f.mean(axis=(2, 3)) for f in feats], axis=1)
    logits = feat @ units[2].w.T + units[2].b
    want_correct = int(np.sum(np.argmax(logits, axis=1) == labels))
    m = logits.max(axis=1, keepdims=True)
    ce = np.log(np.exp(logits - m).sum(axis=1)) + m[:, 0] - logits[np.arange(B), labels]
    # the argmax is an integer decided from floating point: it may differ from the fp64
    # reference only on rows whose top two logits lie within the arithmetic's error
    srt = np.sort(logits, axis=1)
    band = (1e-5 if precision == L.FP32 else 5e-2) * np.abs(logits).max()
    ambiguous = int(np.sum(srt[:, -1] - srt[:, -2] < band))
    assert abs(correct.item() - 2 * want_correct) <= 2 * ambiguous
    assert abs(loss.item() - ce.mean()) <= (1e-4 if precision == L.FP32 else 2e-2) * abs(ce.mean())
    after = st.get_params()
    for a, b in zip(before, after):
        assert np.array_equal(a, b)
    st.close()
