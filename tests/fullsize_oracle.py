"""Oracle side of the full-size single-tick parity tests (test infrastructure).

One micro-batch of the benchmark workload (RevNet-18, CIFAR-10 shape, batch 64,
J = 4, partition [5,4,4,5]; BASELINE.json configs[1], bench.py's default) is pushed
through the EXACT fp64 oracle stage by stage -- every stage's forward, the tail
step, then every stage's backward -- which fixes each stage's inputs:

    x_in[j]            the forward message stage j receives (stage 1: the image)
    xt_out[j], d_out[j] the backward message it receives from stage j+1

Every stage is then a state-injected single tick on those inputs (PAPER.md:131-135:
forward at theta^t, reconstruction + VJP at theta^t, immediate update), run by
  * "exact"   -- the fp64 oracle (the chain itself);
  * "bf16"    -- the oracle under rules R1-R3 (oracle.primitives.bf16_convolutions,
                 DESIGN.md reading c22): conv operands and z rounded to bf16;
  * "pinned"  -- the same bf16 arithmetic with every ReLU mask REPLAYED from the
                 exact run (oracle.primitives.MASKS), i.e. bf16 rounding without its
                 mask flips: the decomposition of reading c25.
No value here comes from the CUDA path; the GPU stage gets the same inputs and
initial state and is compared with these three records.
"""
from __future__ import annotations

import contextlib
import copy
import functools

import numpy as np

import synth
from oracle import engine as E
from oracle import models as OM
from oracle import primitives as OP

WORKLOADS = {
    # name: (model, image, classes, batch, counts, weight decay)
    "r18_b64_j4": ("revnet18", 32, 10, 64, [5, 4, 4, 5], 5e-4),
}
LR = 0.025  # PAPER.md:256, 0.1 * 64 / 256 at k = 1
# the fp32 rounding band of a mask decision (reading c25): 4 sigma of the rounding
# error of a K-term fp32 dot product relative to its rms, u * sqrt(K) with
# u = 2^-24 and K up to 4608 (RevNet's 3x3 x 512): 4 * 6e-8 * 68 = 1.6e-5 -> 2e-5
BAND_FP32 = 2e-5


@contextlib.contextmanager
def oracle_mode(bf16=False, acc32=False, band=None):
    """The oracle's arithmetic for one run: rules R1-R3 (bf16), fp32 rounding (acc32),
    mask decisions in the fp32 band flipped (band)."""
    with contextlib.ExitStack() as st:
        if bf16:
            st.enter_context(OP.bf16_convolutions())
        if acc32:
            st.enter_context(OP.fp32_accumulation())
        prev = OP.MASKS["band"]
        OP.MASKS["band"] = band
        try:
            yield
        finally:
            OP.MASKS["band"] = prev


def init_units(model, H, classes, seed=1):
    """The benchmark's architecture with harness parameters: Kaiming-uniform weights,
    gamma / beta perturbed from (1, 0) so BN is not the identity (reading c17)."""
    units = OM.init_params(OM.build_revnet(model, H, classes), seed)
    i = 0
    for u in units:
        for name, p, _ in u.params():
            if name == "gamma":
                p[...] = 1.0 + 0.2 * synth.normal(p.shape, seed, 100, i)
            elif name in ("beta", "b"):
                p[...] = 0.1 * synth.normal(p.shape, seed, 101, i)
            i += 1
    return units


def _snap(stage):
    return {"theta": [p.copy() for (_, p, _) in stage.params()],
            "v": [v.copy() for v in stage.v],
            "buffers": [b.copy() for (_, b) in stage.buffers()],
            "grads": [g.copy() for g in stage.last_grads]}


def _tick(stage, j, J, x_in, labels, xt, d, masks=None):
    """One forward + one backward of stage j (or the tail step) on the given inputs.
    masks: None, or ("record", dict) / ("replay", dict) with keys "fwd" / "bwd"."""
    rec = {}

    def arm(kind):
        OP.MASKS["record"] = OP.MASKS["replay"] = None
        if masks is None:
            return
        mode, store = masks
        if mode == "record":
            store[kind] = []
            OP.MASKS["record"] = store[kind]
        else:
            OP.MASKS["replay"] = list(store[kind])

    try:
        if j == J:
            arm("fwd")
            loss, bo = stage.tail_step(E.Fwd(0, x_in, labels))
            rec.update(loss=loss, fwd=None, xt=bo.xs, d=bo.ds)
        else:
            arm("fwd")
            fo = stage.forward(E.Fwd(0, x_in, labels))
            arm("bwd")
            bo = stage.backward(E.Bwd(0, xt, d))
            rec.update(loss=None, fwd=fo.xs, xt=bo.xs, d=bo.ds)
    finally:
        OP.MASKS["record"] = OP.MASKS["replay"] = None
    rec.update(_snap(stage))
    return rec


@functools.lru_cache(maxsize=None)
def chain(workload="r18_b64_j4"):
    """Returns (units0, counts, inputs, records) where records[mode][j] is the
    single-tick record of stage j in that mode and inputs[j] = (x_in, labels, xt, d).
    units0 is an untouched copy of the initial parameters (for the GPU stage)."""
    model, H, classes, B, counts, wd = WORKLOADS[workload]
    opt = E.OptConfig(weight_decay=wd)
    units0 = init_units(model, H, classes)
    J = len(counts)
    x0 = [synth.images((B, 3, H, H), 0, 0)]
    lab = synth.labels(B, classes, 0, 0)

    # exact chain: forwards, tail, backwards (records the exact masks per stage)
    units = copy.deepcopy(units0)
    stages = [E.Stage(g, opt, j + 1, J) for j, g in enumerate(OM.group(units, counts))]
    for s in stages:
        s.lr = LR
    masks = {j: {} for j in range(1, J + 1)}
    x_in = {1: x0}
    fwd_out = {}
    for j in range(1, J):
        OP.MASKS["record"] = masks[j].setdefault("fwd", [])
        fwd_out[j] = stages[j - 1].forward(E.Fwd(0, x_in[j], lab)).xs
        OP.MASKS["record"] = None
        x_in[j + 1] = fwd_out[j]
    recs = {"exact": {}}
    OP.MASKS["record"] = masks[J].setdefault("fwd", [])
    loss, bo = stages[J - 1].tail_step(E.Fwd(0, x_in[J], lab))
    OP.MASKS["record"] = None
    recs["exact"][J] = dict(loss=loss, fwd=None, xt=bo.xs, d=bo.ds, **_snap(stages[J - 1]))
    bwd_in = {J - 1: (bo.xs, bo.ds)}
    for j in range(J - 1, 0, -1):
        xt, d = bwd_in[j]
        OP.MASKS["record"] = masks[j].setdefault("bwd", [])
        b = stages[j - 1].backward(E.Bwd(0, xt, d))
        OP.MASKS["record"] = None
        recs["exact"][j] = dict(loss=None, fwd=fwd_out[j], xt=b.xs, d=b.ds, **_snap(stages[j - 1]))
        if j > 1:
            bwd_in[j - 1] = (b.xs, b.ds)
    inputs = {j: (x_in[j], lab, *(bwd_in[j] if j < J else (None, None))) for j in range(1, J + 1)}

    # the other oracle runs, stage by stage on the same inputs (masks recorded, or
    # replayed for "pinned"):
    #   bf16         rules R1-R3                         (the bf16 path's arithmetic)
    #   pinned       rules R1-R3 with the exact masks     (c25: the floor is the flips)
    #   *_acc32      convolutions accumulated / tensors stored in fp32 (c25: another rounding)
    #   *_band       every decision within the fp32 rounding band of zero flipped (c25)
    runs = {"bf16": (True, False, None), "pinned": (True, False, None), "exact_acc32": (False, True, None),
            "bf16_acc32": (True, True, None), "exact_band": (False, False, BAND_FP32),
            "bf16_band": (True, False, BAND_FP32)}
    mrec = {m: {j: {} for j in range(1, J + 1)} for m in runs}
    for mode, (b16, a32, band) in runs.items():
        recs.setdefault(mode, {})
        units = copy.deepcopy(units0)
        groups = OM.group(units, counts)
        for j in range(1, J + 1):
            s = E.Stage(groups[j - 1], opt, j, J)
            s.lr = LR
            m = ("replay", masks[j]) if mode == "pinned" else ("record", mrec[mode][j])
            with oracle_mode(b16, a32, band):
                recs[mode][j] = _tick(s, j, J, *inputs[j], masks=m)
    mrec["exact"] = masks

    def count(a, b):
        out = {}
        for j in range(1, J + 1):
            f = n = 0
            for kind in mrec[a][j]:
                for x, y in zip(mrec[a][j][kind], mrec[b][j][kind]):
                    f += int(np.count_nonzero(x != y))
                    n += x.size
            out[j] = (f, n)
        return out

    # mask decisions that differ, per stage: (flipped, total)
    flips = {"bf16_vs_exact": count("bf16", "exact"), "exact_acc32_vs_exact": count("exact_acc32", "exact"),
             "bf16_acc32_vs_bf16": count("bf16_acc32", "bf16"), "exact_band_vs_exact": count("exact_band", "exact"),
             "bf16_band_vs_bf16": count("bf16_band", "bf16")}
    return units0, counts, inputs, recs, flips
