"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
identical seeded inputs and parameters.  Tolerances (north_star): rel 1e-4 for
the fp32 path, rel 2e-2 for the bf16 tensor-core path (tests/parity_rule.py),
integer schedule reports bit-exact."""

import numpy as np
import pytest

import synth
from oracle import engine as E
from oracle import models as OM
from oracle.units import Branch, ConvBN, DSUnit, RevUnit, StemUnit, TailUnit
from tests.gpu_harness import (nchw, nhwc, oracle_to_product_units, pack_like, pack_params, per_tensor_rel,
                               rand_params, rel)
from tests import fullsize_oracle as FO
from tests.parity_rule import Report

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2406_02052_b200 import Pipeline, Stage  # noqa: E402
from paper_2406_02052_b200 import _lib as L  # noqa: E402
from paper_2406_02052_b200 import models as PM  # noqa: E402

# Comparison rule: tests/parity_rule.py (fp32 vs the exact oracle 1e-4; bf16 vs the
# oracle under rules R1-R3 2e-2, and vs the exact oracle 2e-2 / floor + 2e-2 for
# mask-gated tensors, readings c22 and c25).


@pytest.fixture(scope="module", autouse=True)
def cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    L.lib()


def dev(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def rev(c, dst, k=3):
    return RevUnit(dst, Branch([ConvBN(c, c, k, 1)]))


def bott(c, mid, dst):
    return RevUnit(dst, Branch([ConvBN(c, mid, 1, 1), ConvBN(mid, mid, 3, 1), ConvBN(mid, c, 1, 1)]))


def ds_basic(ci, co, s=2):
    return DSUnit(0, Branch([ConvBN(ci, co, 3, s)]), ConvBN(ci, co, 1, s, relu=False),
                  ConvBN(ci, co, 1, s, relu=False))


def ds_bott(ci, mid, co, s=2):
    return DSUnit(0, Branch([ConvBN(ci, mid, 1, 1), ConvBN(mid, mid, 3, s), ConvBN(mid, co, 1, 1)]),
                  ConvBN(ci, co, 1, s, relu=False), ConvBN(ci, co, 1, s, relu=False))


def make_pair(units, B, in_hwc, precision, seed=3):
    rand_params(units, seed)
    spec = PM.StageSpec(oracle_to_product_units(units), B, in_hwc, precision, fifo_capacity=3)
    st = Stage(spec, seed=0)
    th, bf = pack_params(units)
    assert th.size == st.n_params and bf.size == st.n_buffers
    st.set_params(th, np.zeros_like(th), bf)
    return st


def check(name, got, want, tol, report):
    r = rel(got, want)
    report.append((name, r))
    return r <= tol


STAGE_CASES = {
    # name: (units factory, batch, input NCHW shapes)
    "rev_basic_c64_32x32": (lambda: [rev(64, 0), rev(64, 1)], 2, [(2, 64, 32, 32)] * 2),
    "rev_basic_c128_16x16": (lambda: [rev(128, 0), rev(128, 1)], 2, [(2, 128, 16, 16)] * 2),
    "rev_bottleneck": (lambda: [bott(64, 16, 0), bott(64, 16, 1)], 4, [(4, 64, 8, 8)] * 2),
    "ds_basic_then_rev": (lambda: [ds_basic(32, 64), rev(64, 1)], 4, [(4, 32, 16, 16)] * 2),
    "ds_bottleneck_then_rev": (lambda: [ds_bott(32, 16, 64), bott(64, 16, 1)], 2, [(2, 32, 12, 12)] * 2),
    "rev_then_ds": (lambda: [rev(32, 1), ds_basic(32, 64), rev(64, 1)], 2, [(2, 32, 8, 8)] * 2),
    "stem_cifar_then_rev": (lambda: [StemUnit(3, 64, 3, 1, False), rev(32, 0)], 4, [(4, 3, 16, 16)]),
    "stem_imagenet_maxpool": (lambda: [StemUnit(3, 32, 7, 2, True), rev(16, 0)], 2, [(2, 3, 30, 30)]),
    # ResNet-50 grids with padded tensor-core tiles (14 -> Wb 16, 7 -> Wb 8, odd batch)
    "r50_bottleneck_single_14x14": (lambda: [bott(128, 64, 1)], 2, [(2, 128, 14, 14)] * 2),
    "r50_ds_bottleneck_single_14_to_7": (lambda: [ds_bott(128, 64, 256)], 3, [(3, 128, 14, 14)] * 2),
    "r50_bottleneck_14x14": (lambda: [bott(128, 64, 0), bott(128, 64, 1)], 2, [(2, 128, 14, 14)] * 2),
    "r50_ds_bottleneck_14_to_7": (lambda: [ds_bott(128, 64, 256), bott(256, 64, 1)], 3, [(3, 128, 14, 14)] * 2),
}


def _oracle_stage_tick(make, B, in_shapes, bf16, acc32=False, band=None):
    """The oracle's single tick of a non-final stage on the test's inputs."""
    units = make()
    rand_params(units, 3)
    ostage = E.Stage(units, E.OptConfig(), 1, 2)
    ostage.lr = 0.1
    xs = [synth.images(s, 0, i) for i, s in enumerate(in_shapes)]
    # backward on a received (x~, delta): the EXACT forward output perturbed (the same
    # message for both oracles and the GPU), random delta
    xt = [a + 0.05 * synth.normal(a.shape, 7, h) for h, a in enumerate(_exact_fwd(make, B, in_shapes))]
    dd = [synth.normal(a.shape, 8, h) for h, a in enumerate(xt)]
    with FO.oracle_mode(bf16, acc32, band):
        fo = ostage.forward(E.Fwd(0, xs, None))
        bo = ostage.backward(E.Bwd(0, xt, dd))
    th, bf = pack_params(units)
    return {"units": units, "xs": xs, "fwd": fo.xs, "xt_in": xt, "d_in": dd, "xt": bo.xs, "d": bo.ds,
            "grads": pack_like(units, ostage.last_grads), "theta": th, "v": pack_like(units, ostage.v),
            "buffers": bf}


_FWD_CACHE = {}


def _exact_fwd(make, B, in_shapes):
    key = (make, B, tuple(map(tuple, in_shapes)))
    if key not in _FWD_CACHE:
        units = make()
        rand_params(units, 3)
        xs = [synth.images(s, 0, i) for i, s in enumerate(in_shapes)]
        _FWD_CACHE[key] = E.Stage(units, E.OptConfig(), 1, 2).forward(E.Fwd(0, xs, None)).xs
    return _FWD_CACHE[key]


def _slices(units):
    out, off = [], 0
    for ui, u in enumerate(units):
        for name, p, _ in u.params():
            out.append((f"u{ui}.{name}", off, off + p.size))
            off += p.size
    return out


@pytest.mark.parametrize("precision", [L.FP32, L.BF16_TC], ids=["fp32", "bf16"])
@pytest.mark.parametrize("case", sorted(STAGE_CASES))
def test_stage_tick_parity(case, precision):
    """One forward tick then one backward tick (reconstruction with the current
    theta + VJP + immediate Nesterov update) of a non-final stage."""
    make, B, in_shapes = STAGE_CASES[case]
    bf16 = precision == L.BF16_TC
    ex = _oracle_stage_tick(make, B, in_shapes, False)
    bq = _oracle_stage_tick(make, B, in_shapes, True) if bf16 else None
    alts = [_oracle_stage_tick(make, B, in_shapes, bf16, acc32=True),
            _oracle_stage_tick(make, B, in_shapes, bf16, band=FO.BAND_FP32)]
    units = make()
    stem = isinstance(units[0], StemUnit)
    in_hwc = tuple(np.array(in_shapes[0])[[2, 3, 1]])
    st = make_pair(units, B, in_hwc, precision)
    rep = Report(bf16)
    b_ = (lambda k, i=None: (bq[k] if i is None else bq[k][i]) if bf16 else None)
    Bq, Ho, Wo, Co = st.out_shape
    o = [torch.empty((Bq, Ho, Wo, Co), device="cuda") for _ in range(2)]
    gx = [dev(nhwc(x)) for x in ex["xs"]]
    st.forward(0, gx[0], gx[1] if not stem else None, o[0], o[1])
    torch.cuda.synchronize()
    for h in range(2):
        rep.add(f"fwd.x{h + 1}", nchw(host(o[h])), ex["fwd"][h], b_("fwd", h))
    in_half = [torch.empty((B,) + tuple(in_hwc[:2]) + (in_hwc[2],), device="cuda") for _ in range(4)]
    gxt, gd = [dev(nhwc(x)) for x in ex["xt_in"]], [dev(nhwc(d)) for d in ex["d_in"]]
    if stem:
        st.backward(0, gxt[0], gxt[1], gd[0], gd[1], None, None, None, None, 0.1)
    else:
        st.backward(0, gxt[0], gxt[1], gd[0], gd[1], *in_half, 0.1)
    torch.cuda.synchronize()
    if not stem:
        for h in range(2):
            rep.add(f"bwd.xt{h + 1}", nchw(host(in_half[h])), ex["xt"][h], b_("xt", h))
            rep.add(f"bwd.d{h + 1}", nchw(host(in_half[2 + h])), ex["d"][h], b_("d", h), gated=True,
                    alt=[a["d"][h] for a in alts])
    g = st.get_grads()
    th, v, bf = st.get_params()
    for name, a, b in _slices(units):
        for key, got in (("grads", g), ("theta", th), ("v", v)):
            rep.add(f"{key}.{name}", got[a:b], ex[key][a:b], bq[key][a:b] if bf16 else None, gated=True,
                    alt=[x[key][a:b] for x in alts])
    rep.add("running", bf, ex["buffers"], b_("buffers"))
    print(rep.text())
    assert rep.ok, "\n" + rep.text()


TAIL_CASES = {
    "rev_rev_tail": (lambda: [rev(32, 0), rev(32, 1), TailUnit(64, 10)], 8, [(8, 32, 8, 8)] * 2),
    "ds_rev_tail": (lambda: [ds_basic(16, 32), rev(32, 1), TailUnit(64, 10)], 4, [(4, 16, 8, 8)] * 2),
    "bottleneck_tail_1000": (lambda: [bott(64, 16, 0), TailUnit(128, 1000)], 4, [(4, 64, 4, 4)] * 2),
    # a reversible unit BEFORE a downsampling unit in the final stage (RevNet-50 J=4's last stage)
    "rev_ds_rev_tail": (lambda: [rev(16, 1), ds_basic(16, 32), rev(32, 1), TailUnit(64, 10)], 4, [(4, 16, 8, 8)] * 2),
    # tensor-core geometries (channels multiples of 64) for the bf16 path
    "tc_ds_rev_tail": (lambda: [ds_basic(64, 128), rev(128, 1), TailUnit(256, 10)], 8, [(8, 64, 16, 16)] * 2),
    "tc_bottleneck_tail_1000": (lambda: [bott(256, 64, 0), bott(256, 64, 1), TailUnit(512, 1000)], 4,
                                [(4, 256, 7, 7)] * 2),
}


def _oracle_tail(make, B, in_shapes, bf16, acc32=False, band=None):
    units = make()
    rand_params(units, 3)
    ostage = E.Stage(units, E.OptConfig(), 2, 2)
    ostage.lr = 0.1
    xs = [synth.images(s, 0, i) for i, s in enumerate(in_shapes)]
    lab = synth.labels(B, units[-1].classes, 0, 0)
    with FO.oracle_mode(bf16, acc32, band):
        loss, bo = ostage.tail_step(E.Fwd(0, xs, lab))
    th, bf = pack_params(units)
    return {"xs": xs, "lab": lab, "loss": loss, "d": bo.ds, "grads": pack_like(units, ostage.last_grads),
            "theta": th, "v": pack_like(units, ostage.v), "buffers": bf}


@pytest.mark.parametrize("precision", [L.FP32, L.BF16_TC], ids=["fp32", "bf16"])
@pytest.mark.parametrize("case", sorted(TAIL_CASES))
def test_tail_stage_parity(case, precision):
    """Final stage: forward with stored graph, loss, backprop, update (reading c7/c10)."""
    make, B, in_shapes = TAIL_CASES[case]
    bf16 = precision == L.BF16_TC
    ex = _oracle_tail(make, B, in_shapes, False)
    bq = _oracle_tail(make, B, in_shapes, True) if bf16 else None
    alts = [_oracle_tail(make, B, in_shapes, bf16, acc32=True),
            _oracle_tail(make, B, in_shapes, bf16, band=FO.BAND_FP32)]
    units = make()
    in_hwc = tuple(np.array(in_shapes[0])[[2, 3, 1]])
    st = make_pair(units, B, in_hwc, precision)
    gx = [dev(nhwc(x)) for x in ex["xs"]]
    outs = [torch.empty_like(gx[0]) for _ in range(4)]
    loss = torch.zeros(1, device="cuda")
    st.tail(0, gx[0], gx[1], dev(ex["lab"], torch.int32), 0.1, *outs, loss)
    torch.cuda.synchronize()
    rep = Report(bf16)
    rep.add("loss", [loss.item()], [ex["loss"]], [bq["loss"]] if bf16 else None, tol=None if bf16 else 1e-5)
    for h in range(2):
        # the tail returns the received input unchanged (reading c7): bit-exact copy
        rep.add(f"xt{h + 1}", nchw(host(outs[h])), ex["xs"][h].astype(np.float32),
                ex["xs"][h].astype(np.float32) if bf16 else None, tol=0.0)
        rep.add(f"d{h + 1}", nchw(host(outs[2 + h])), ex["d"][h], bq["d"][h] if bf16 else None, gated=True,
                alt=[a["d"][h] for a in alts])
    g = st.get_grads()
    th, v, bf = st.get_params()
    for name, a, b in _slices(units):
        for key, got in (("grads", g), ("theta", th), ("v", v)):
            rep.add(f"{key}.{name}", got[a:b], ex[key][a:b], bq[key][a:b] if bf16 else None, gated=True,
                    alt=[x[key][a:b] for x in alts])
    rep.add("running", bf, ex["buffers"], bq["buffers"] if bf16 else None)
    print(rep.text())
    assert rep.ok, "\n" + rep.text()


def run_pipeline_pair(o_units, counts, B, image_nchw, classes, n_mb, lr, drain, precision=L.FP32,
                      rev_first=False, k=1):
    rand_params(o_units, 5)
    groups = OM.group(o_units, counts)
    init = [pack_params(g) for g in groups]   # before the oracle trains them
    ost = [E.Stage(g, E.OptConfig(k=k)) for g in groups]

    def batch_fn(m):
        x = synth.images(image_nchw, 0, m)
        y = synth.labels(B, classes, 0, m)
        if rev_first:
            h = image_nchw[1] // 2
            return [x[:, :h].copy(), x[:, h:].copy()], y
        return [x], y

    reps, losses, _ = E.run_petra(ost, batch_fn, n_mb, lr=lr, drain=drain)
    p_units = oracle_to_product_units(o_units)
    hwc = (image_nchw[2], image_nchw[3], image_nchw[1] // 2 if rev_first else image_nchw[1])
    specs = PM.stage_specs(p_units, counts, B, hwc, precision, accumulation_k=k)
    pipe = Pipeline(specs, seed=0)
    for j, (th, bf) in enumerate(init, 1):
        pipe.stages[j].set_params(th, np.zeros_like(th), bf)
    loss = torch.zeros(1, device="cuda")
    g_reps, g_losses = [], {}
    for t in range(len(reps)):
        inject = t < n_mb
        x0 = lab = None
        if inject:
            xs, y = batch_fn(t)
            x0 = dev(np.concatenate([nhwc(x).ravel() for x in xs]))
            lab = dev(y, torch.int32)
        loss.fill_(float("nan"))
        r = pipe.tick(t, inject, x0, lab, lr, loss)
        torch.cuda.synchronize()
        g_reps.append(r)
        if r["fwd_mb"][-1] >= 0:
            g_losses[r["fwd_mb"][-1]] = loss.item()
    return reps, losses, ost, groups, pipe, g_reps, g_losses


def compare_pipeline(reps, losses, ost, groups, pipe, g_reps, g_losses, tol, v_tol=None):
    for r, g in zip(reps, g_reps):   # integer report: bit-exact
        assert g["fwd_mb"] == r.fwd_mb and g["bwd_mb"] == r.bwd_mb, (r, g)
        assert g["version"] == r.version and g["fifo_depth"] == r.fifo_depth, (r, g)
    assert sorted(g_losses) == sorted(losses)
    errs = {f"loss{m}": abs(g_losses[m] - losses[m]) / abs(losses[m]) for m in losses}
    for j, (s, g) in enumerate(zip(ost, groups), 1):
        th, v, _ = pipe.stages[j].get_params()
        want, _ = pack_params(g)
        errs[f"theta{j}"] = rel(th, want)
        errs[f"v{j}"] = rel(v, pack_like(g, s.v))
    print("pipeline parity:", ", ".join(f"{k} {v:.2e}" for k, v in errs.items()))
    bad = {k: e for k, e in errs.items() if e > (v_tol if (k.startswith("v") and v_tol) else tol)}
    assert not bad, bad


@pytest.mark.parametrize("k", [1, 2, 3])
def test_pipeline_mlp_config1(k):
    """Config 1 (reading c16): 2-stage reversible MLP, d=64, batch 32, 10 ticks, fp32;
    k > 1 = gradient accumulation (Alg. 1 lines 19-23): updates on
    every k-th backward with the average Delta, version = floor(n_bwd / k) bit-exact."""
    units = OM.build_mlp(64, 10)
    out = run_pipeline_pair(units, [2, 3], 32, (32, 64, 1, 1), 10, 10, 0.025 * k, drain=False, rev_first=True,
                            k=k)
    compare_pipeline(*out, tol=1e-4)


@pytest.mark.parametrize("k", [2, 4])
def test_pipeline_revnet18_accumulation(k):
    """RevNet-18 J=4 with accumulation k: 6 micro-batches plus
    drain, free-running, fp32; integers bit-exact, losses 1e-4.  Parameters: the
    trajectory is free-running, so a ReLU mask whose pre-activation lies within the
    ~1e-6 fp32 drift of the messages can flip (reading c20) and every update after
    it carries the flip: theta is held to 2e-4 and the momentum buffers to 2e-2
    (measured theta1 1.5e-4 at k = 2, lr 0.02).  The accumulate / update arithmetic
    itself is held to 1e-4 by test_pipeline_mlp_config1[k]."""
    units = OM.build_revnet("revnet18", 32, 10)
    out = run_pipeline_pair(units, [5, 4, 4, 5], 4, (4, 3, 32, 32), 10, 6, 0.01, drain=True, k=k)
    compare_pipeline(*out, tol=2e-4, v_tol=2e-2)


@pytest.mark.parametrize("lr", [0.0, 0.01])
def test_pipeline_revnet18_cifar_j4(lr):
    """Config 2 architecture (RevNet-18, 32x32, J=4) at batch 4: 4 micro-batches
    plus drain, free-running PETRA schedule, fp32.  Integer reports bit-exact,
    losses and theta at 1e-4.  Momentum buffers integrate every gradient and a
    free-running run may flip a ReLU mask whose pre-activation lies within the
    ~1e-6 fp32 drift of the messages (reading c20), so they are held to 2e-2
    here; test_free_running_stages_vs_oracle_on_gpu_messages checks each
    backward strictly on the GPU's own messages."""
    units = OM.build_revnet("revnet18", 32, 10)
    out = run_pipeline_pair(units, [5, 4, 4, 5], 4, (4, 3, 32, 32), 10, 4, lr, drain=True)
    compare_pipeline(*out, tol=1e-4, v_tol=2e-2)


def stage_loop(specs, init, fn, n_mb, lr, J, B, on_backward=None):
    """Free-running PETRA schedule over standalone GPU stages with Python
    double-buffered mailboxes (the reference for the Pipeline's bookkeeping)."""
    gst = [Stage(s, 0) for s in specs]
    for s, (th, bf) in zip(gst, init):
        s.set_params(th, np.zeros_like(th), bf)
    gf, gb, losses = [None] * (J + 2), [None] * (J + 2), {}
    for t in range(n_mb + 2 * J - 2):
        nf, nb = [None] * (J + 2), [None] * (J + 2)
        for j in range(1, J + 1):
            g = gst[j - 1]
            if j == 1:
                fin = None
                if t < n_mb:
                    xs, y = fn(t)
                    fin = (t, [dev(nhwc(xs[0])), None], dev(y, torch.int32))
            else:
                fin = gf[j]
            shp = (B,) + tuple(specs[j - 1].in_shape)
            if j < J:
                if fin is not None:
                    o = [torch.empty(g.out_shape, device="cuda") for _ in range(2)]
                    g.forward(fin[0], fin[1][0], fin[1][1], o[0], o[1])
                    nf[j + 1] = (fin[0], o, fin[2])
                if gb[j] is not None:
                    mb, msg = gb[j]
                    res = [torch.empty(shp, device="cuda") for _ in range(4)] if j > 1 else [None] * 4
                    if on_backward:
                        on_backward(t, j, mb, msg, "before")
                    g.backward(mb, *msg, *res, lr)
                    if on_backward:
                        on_backward(t, j, mb, g, "after")
                    if j > 1:
                        nb[j - 1] = (mb, res)
            elif fin is not None:
                res = [torch.empty(shp, device="cuda") for _ in range(4)]
                loss = torch.zeros(1, device="cuda")
                g.tail(fin[0], fin[1][0], fin[1][1], fin[2], lr, *res, loss)
                nb[j - 1] = (fin[0], res)
                losses[fin[0]] = loss
        gf, gb = nf, nb
    torch.cuda.synchronize()
    return gst, {m: l.item() for m, l in losses.items()}


def test_pipeline_bitwise_equals_stage_loop():
    """The Pipeline object (C++ mailboxes, schedule) is bitwise identical to the
    same stages driven by a Python double-buffered loop (deterministic kernels)."""
    units = rand_params(OM.build_revnet("revnet18", 32, 10), 5)
    counts, B, lr, n_mb, J = [5, 4, 4, 5], 4, 0.025, 5, 4
    groups = OM.group(units, counts)
    init = [pack_params(g) for g in groups]
    specs = PM.stage_specs(oracle_to_product_units(units), counts, B, (32, 32, 3))
    fn = lambda m: ([synth.images((B, 3, 32, 32), 0, m)], synth.labels(B, 10, 0, m))
    gst, losses = stage_loop(specs, init, fn, n_mb, lr, J, B)
    pipe = Pipeline(specs, seed=0)
    for j, (th, bf) in enumerate(init, 1):
        pipe.stages[j].set_params(th, np.zeros_like(th), bf)
    loss = torch.zeros(1, device="cuda")
    plosses = {}
    for t in range(n_mb + 2 * J - 2):
        x0 = lab = None
        if t < n_mb:
            xs, y = fn(t)
            x0, lab = dev(nhwc(xs[0])), dev(y, torch.int32)
        r = pipe.tick(t, t < n_mb, x0, lab, lr, loss)
        if r["fwd_mb"][-1] >= 0:
            plosses[r["fwd_mb"][-1]] = loss.item()
    assert plosses == losses
    for j in range(1, J + 1):
        a, b = pipe.stages[j].get_params(), gst[j - 1].get_params()
        for x, y in zip(a, b):
            assert np.array_equal(x, y), j


def test_free_running_stages_vs_oracle_on_gpu_messages():
    """Every backward of a free-running GPU pipeline (RevNet-18, J=4, lr>0)
    against a copy of the oracle stage in the same state fed the GPU's OWN
    message (x~, delta): rel 1e-4 per tensor.  Together with the stage-level
    tests this pins each tick; the oracle's own free-running trajectory may
    differ by ReLU-mask flips (reading c20)."""
    units = rand_params(OM.build_revnet("revnet18", 32, 10), 5)
    counts, B, lr, n_mb, J = [5, 4, 4, 5], 4, 0.025, 4, 4
    groups = OM.group(units, counts)
    init = [pack_params(g) for g in groups]
    ost = [E.Stage(g, E.OptConfig()) for g in groups]
    for j, s in enumerate(ost, 1):
        s.j, s.J = j, J
    specs = PM.stage_specs(oracle_to_product_units(units), counts, B, (32, 32, 3))
    fn = lambda m: ([synth.images((B, 3, 32, 32), 0, m)], synth.labels(B, 10, 0, m))
    worst = {}

    def H(t):
        return nchw(t.detach().cpu().numpy().astype(np.float64))

    # run the GPU loop; before each GPU backward the oracle copy of that stage runs
    # its backward on the GPU message (the oracle copy is advanced in lockstep)
    gst = [Stage(s, 0) for s in specs]
    for s, (th, bf) in zip(gst, init):
        s.set_params(th, np.zeros_like(th), bf)
    gf, gb = [None] * (J + 2), [None] * (J + 2)
    for t in range(n_mb + 2 * J - 2):
        nf, nb = [None] * (J + 2), [None] * (J + 2)
        for j in range(1, J + 1):
            g, s = gst[j - 1], ost[j - 1]
            s.lr = lr
            if j == 1:
                fin = None
                if t < n_mb:
                    xs, y = fn(t)
                    fin = (t, [dev(nhwc(xs[0])), None], dev(y, torch.int32), xs, y)
            else:
                fin = gf[j]
            shp = (B,) + tuple(specs[j - 1].in_shape)
            if j < J:
                if fin is not None:
                    o = [torch.empty(g.out_shape, device="cuda") for _ in range(2)]
                    g.forward(fin[0], fin[1][0], fin[1][1], o[0], o[1])
                    oxs = fin[3] if j == 1 else [H(fin[1][0]), H(fin[1][1])]
                    s.forward(E.Fwd(fin[0], oxs, fin[4]))          # oracle FIFO gets the GPU input
                    nf[j + 1] = (fin[0], o, fin[2], None, fin[4])
                if gb[j] is not None:
                    mb, msg = gb[j]
                    om = E.Bwd(mb, [H(msg[0]), H(msg[1])], [H(msg[2]), H(msg[3])])
                    s.backward(om)   # oracle stage holds the GPU stage's theta / v (synced)
                    res = [torch.empty(shp, device="cuda") for _ in range(4)] if j > 1 else [None] * 4
                    g.backward(mb, *msg, *res, lr)
                    torch.cuda.synchronize()
                    errs = per_tensor_rel(groups[j - 1], g.get_grads(), pack_like(groups[j - 1], s.last_grads))
                    worst[(t, j, mb)] = max(e for _, e in errs)
                    # re-sync the oracle stage's theta/v to the GPU's (removes drift)
                    _sync_oracle_stage(s, groups[j - 1], g)
                    if j > 1:
                        nb[j - 1] = (mb, res)
            elif fin is not None:
                res = [torch.empty(shp, device="cuda") for _ in range(4)]
                loss = torch.zeros(1, device="cuda")
                g.tail(fin[0], fin[1][0], fin[1][1], fin[2], lr, *res, loss)
                torch.cuda.synchronize()
                s.tail_step(E.Fwd(fin[0], [H(fin[1][0]), H(fin[1][1])], fin[4]))
                errs = per_tensor_rel(groups[j - 1], g.get_grads(), pack_like(groups[j - 1], s.last_grads))
                worst[(t, j, fin[0])] = max(e for _, e in errs)
                _sync_oracle_stage(s, groups[j - 1], g)
                nb[j - 1] = (fin[0], res)
        gf, gb = nf, nb
    # isolated ReLU-mask flips (a pre-activation within the fp32/fp64 forward
    # difference of 0) are the expected outliers (reading c20): at most 10% of
    # the backward events may exceed 1e-4, none may exceed 2e-2
    assert len(worst) == 4 * n_mb
    print("per-backward max rel:", {k: f"{v:.1e}" for k, v in sorted(worst.items())})
    outliers = {k: v for k, v in worst.items() if v > 1e-4}
    assert len(outliers) <= 0.1 * len(worst) and max(worst.values()) <= 2e-2, outliers


def _sync_oracle_stage(s, units, g):
    """Copy the GPU stage's theta / v into the oracle stage (layout inverse of pack)."""
    th, v, _ = g.get_params()
    off = 0
    for (name, p, _), vv in zip(s.params(), s.v):
        n = p.size
        for src, dst in ((th, p), (v, vv)):
            a = src[off:off + n].astype(np.float64)
            if name == "w" and p.ndim == 4:
                co, ci, k, _ = p.shape
                a = a.reshape(co, k, k, ci).transpose(0, 3, 1, 2)
            dst[...] = a.reshape(p.shape)
        off += n


@pytest.mark.parametrize("case", ["ds_basic_then_rev", "stem_cifar_then_rev", "rev_basic_c64_32x32"])
def test_stage_fifo_depth3(case):
    """Three forwards in flight before the backwards (FIFO depth 3, as at stage
    J-1 of a J=2.5 pipeline), lr=0 so the oracle's theta is fixed: every
    backward must match the oracle on the same (x~, delta)."""
    make, B, in_shapes = STAGE_CASES[case]
    units = make()
    stem = isinstance(units[0], StemUnit)
    in_hwc = tuple(np.array(in_shapes[0])[[2, 3, 1]])
    st = make_pair(units, B, in_hwc, L.FP32)
    ostage = E.Stage(units, E.OptConfig(), 1, 3)
    ostage.lr = 0.0
    rep, ok = [], True
    outs = []
    for m in range(3):
        xs = [synth.images(s, 10 + m, i) for i, s in enumerate(in_shapes)]
        fo = ostage.forward(E.Fwd(m, xs, None))
        o = [torch.empty(st.out_shape, device="cuda") for _ in range(2)]
        gx = [dev(nhwc(x)) for x in xs]
        st.forward(m, gx[0], gx[1] if not stem else None, o[0], o[1])
        outs.append((fo, o))
    for m in range(3):
        fo, o = outs[m]
        dd = [synth.normal(fo.xs[h].shape, 20 + m, h) for h in range(2)]
        bo = ostage.backward(E.Bwd(m, fo.xs, dd))
        res = [torch.empty((B,) + tuple(in_hwc), device="cuda") for _ in range(4)]
        gxt = [dev(nhwc(x)) for x in fo.xs]
        gd = [dev(nhwc(d)) for d in dd]
        st.backward(m, gxt[0], gxt[1], gd[0], gd[1], *(res if not stem else [None] * 4), 0.0)
        torch.cuda.synchronize()
        if not stem:
            for h in range(2):
                ok &= check(f"mb{m}.xt{h}", nchw(host(res[h])), bo.xs[h], 1e-4, rep)
                ok &= check(f"mb{m}.d{h}", nchw(host(res[2 + h])), bo.ds[h], 1e-4, rep)
        for name, r in per_tensor_rel(units, st.get_grads(), pack_like(units, ostage.last_grads)):
            rep.append((f"mb{m}.grad.{name}", r))
            ok &= r <= 1e-4
    assert ok, "\n".join(f"{n}: {r:.3e}" for n, r in rep)


@pytest.mark.parametrize("case", sorted(TAIL_CASES))
def test_tail_stage_consecutive(case):
    """Three consecutive final-stage steps (state carried between calls)."""
    make, B, in_shapes = TAIL_CASES[case]
    units = make()
    in_hwc = tuple(np.array(in_shapes[0])[[2, 3, 1]])
    st = make_pair(units, B, in_hwc, L.FP32)
    ostage = E.Stage(units, E.OptConfig(), 2, 2)
    ostage.lr = 0.05
    rep, ok = [], True
    for m in range(3):
        xs = [synth.images(s, 30 + m, i) for i, s in enumerate(in_shapes)]
        lab = synth.labels(B, units[-1].classes, 0, m)
        loss_o, bo = ostage.tail_step(E.Fwd(m, xs, lab))
        gx = [dev(nhwc(x)) for x in xs]
        outs = [torch.empty_like(gx[0]) for _ in range(4)]
        loss = torch.zeros(1, device="cuda")
        st.tail(m, gx[0], gx[1], dev(lab, torch.int32), 0.05, *outs, loss)
        torch.cuda.synchronize()
        rep.append((f"mb{m}.loss", abs(loss.item() - loss_o) / abs(loss_o)))
        for h in range(2):
            ok &= check(f"mb{m}.d{h}", nchw(host(outs[2 + h])), bo.ds[h], 1e-4, rep)
        for name, r in per_tensor_rel(units, st.get_grads(), pack_like(units, ostage.last_grads)):
            rep.append((f"mb{m}.grad." + name, r))
            ok &= r <= 1e-4
    assert ok, "\n".join(f"{n}: {r:.3e}" for n, r in rep)
