"""PETRA fp64 CPU oracle -- RevNet / MLP builders and contiguous stage grouping.

TEST INFRASTRUCTURE, NOT PRODUCT CODE (see oracle/primitives.py header).

Architecture readings ("the number of channels in each stage is
multiplied by 2 ... the number of parameters stays almost the same"; the
appendix that should define it is empty) -- reading c3:
  * RevNet-18/34: ResNet basic blocks [2,2,2,2]/[3,4,6,3] at half-stream widths
    64/128/256/512; each block is the F/G unit pair with Phi = ONE
    conv3x3-BN-ReLU; the first block of layers 2-4 replaces its F unit with a
    downsampling unit (stride-2 Phi_s and per-half 1x1 projections).
  * RevNet-50: bottleneck blocks [3,4,6,3], mid widths 64..512, half-stream
    widths 256..2048; every block is ONE half-coupling with Phi = the full
    bottleneck (1x1, 3x3, 1x1), consecutive reversible blocks alternating F/G;
    block 0 of every layer is a downsampling unit (stride 1 in layer 1).
  * Stem: 3x3/s1 without max-pool for 32x32 inputs (CIFAR; reading c4 for
    ImageNet32), 7x7/s2 + max-pool for 224x224 inputs; 2*64 output channels.
These give 12,384,872 / 22,493,032 / 30,391,144 parameters on ImageNet
(1000 classes), against the paper's 12.2M / 22.3M / 30.4M (Table 2, PAPER.md:
275, 280, 285).
"""
from __future__ import annotations

import numpy as np

import synth
from .units import Branch, ConvBN, DSUnit, RevUnit, StemUnit, TailUnit

BASIC = {"revnet18": [2, 2, 2, 2], "revnet34": [3, 4, 6, 3]}
BOTTLENECK = {"revnet50": [3, 4, 6, 3]}
WIDTHS = [64, 128, 256, 512]


def build_revnet(name: str, image_size: int = 32, classes: int = 10):
    """Returns the flat unit list [stem, ..., tail] (uninitialised parameters)."""
    units = []
    big = image_size >= 128
    units.append(StemUnit(3, 128, 7 if big else 3, 2 if big else 1, maxpool=big))
    if name in BASIC:
        c_prev = 64
        for li, nblk in enumerate(BASIC[name]):
            c = WIDTHS[li]
            for b in range(nblk):
                if b == 0 and li > 0:
                    units.append(DSUnit(0, Branch([ConvBN(c_prev, c, 3, 2)]),
                                        ConvBN(c_prev, c, 1, 2, relu=False),
                                        ConvBN(c_prev, c, 1, 2, relu=False)))
                else:
                    units.append(RevUnit(0, Branch([ConvBN(c, c, 3, 1)])))
                units.append(RevUnit(1, Branch([ConvBN(c, c, 3, 1)])))
            c_prev = c
        units.append(TailUnit(2 * c_prev, classes))
    elif name in BOTTLENECK:
        c_prev = 64
        for li, nblk in enumerate(BOTTLENECK[name]):
            mid = WIDTHS[li]
            c = 4 * mid
            s = 1 if li == 0 else 2
            units.append(DSUnit(0, Branch([ConvBN(c_prev, mid, 1, 1), ConvBN(mid, mid, 3, s),
                                           ConvBN(mid, c, 1, 1)]),
                                ConvBN(c_prev, c, 1, s, relu=False),
                                ConvBN(c_prev, c, 1, s, relu=False)))
            for b in range(1, nblk):
                dst = (b - 1) % 2
                units.append(RevUnit(dst, Branch([ConvBN(c, mid, 1, 1), ConvBN(mid, mid, 3, 1),
                                                  ConvBN(mid, c, 1, 1)])))
            c_prev = c
        units.append(TailUnit(2 * c_prev, classes))
    else:
        raise ValueError(f"unknown model {name}")
    return units


def build_mlp(d: int = 64, classes: int = 10):
    """Config 1 (reading c16): 2 stages; stage 1 = one F/G unit of
    Linear(d/2 -> d/2, no bias)-BN-ReLU branches; stage 2 = one F/G unit + tail.
    A Linear layer is a 1x1 conv on a [B, C, 1, 1] activation; BN over the batch
    is BN1d."""
    h = d // 2
    mk = lambda dst: RevUnit(dst, Branch([ConvBN(h, h, 1, 1)]))
    return [mk(0), mk(1), mk(0), mk(1), TailUnit(d, classes)]


def paper_stage_counts(name: str):
    """Units per stage when the net is "split to preserve each residual block"
    (PAPER.md:259): stem, one stage per block, tail (the tail is its own stage)."""
    if name in BASIC:
        return [1] + [2] * sum(BASIC[name]) + [1]
    return [1] + [1] * sum(BOTTLENECK[name]) + [1]


def group(units, counts):
    """Contiguous grouping of units into stages (reading c14)."""
    assert sum(counts) == len(units), (counts, len(units))
    out, i = [], 0
    for c in counts:
        out.append(units[i:i + c])
        i += c
    return out


def param_count(units) -> int:
    return int(sum(p.size for u in units for (_, p, _) in u.params()))


def init_params(units, seed: int = 1):
    """Harness initialisation (reading c17) drawn from ``synth``: conv/linear
    weights Kaiming-uniform on fan_in, gamma=1, beta=0, bias=0."""
    idx = 0
    for u in units:
        for name, p, _ in u.params():
            if name == "w":
                fan_in = int(np.prod(p.shape[1:]))
                p[...] = synth.kaiming_uniform(p.shape, fan_in, seed, idx)
            elif name == "gamma":
                p[...] = 1.0
            else:
                p[...] = 0.0
            idx += 1
        for _, b in u.buffers():
            pass
    return units


def stage_shapes(units, x_shapes):
    """Propagate activation shapes (NCHW) through the units; returns per-unit
    input shapes and the final shapes."""
    from . import primitives as P
    shapes = [tuple(s) for s in x_shapes]
    ins = []
    for u in units:
        ins.append(shapes)
        if isinstance(u, StemUnit):
            B, C, H, W = shapes[0]
            l = u.layer
            Ho, Wo = P.conv_out_size(H, l.k, l.stride, l.pad), P.conv_out_size(W, l.k, l.stride, l.pad)
            if u.maxpool:
                Ho, Wo = P.conv_out_size(Ho, 3, 2, 1), P.conv_out_size(Wo, 3, 2, 1)
            shapes = [(B, l.cout // 2, Ho, Wo)] * 2
        elif isinstance(u, DSUnit):
            B, C, H, W = shapes[0]
            Ho, Wo = P.conv_out_size(H, 1, u.pa.stride, 0), P.conv_out_size(W, 1, u.pa.stride, 0)
            shapes = [(B, u.pa.cout, Ho, Wo)] * 2
        elif isinstance(u, TailUnit):
            shapes = [(shapes[0][0], u.classes)]
    return ins, shapes
