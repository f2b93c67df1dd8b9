"""RevNet-18/34/50 and the config-1 MLP as PETRA unit lists (product side), the
contiguous stage partitioner and stage descriptors.

Architecture reading (reading c3; Table 2): channels x2
for the second stream; RevNet-18/34 blocks are F/G pairs of one conv3x3-BN-ReLU
each, the first block of layers 2-4 downsamples (stride-2 Phi_s, per-half 1x1
projections); RevNet-50 blocks are single bottleneck half-couplings alternating
F/G, every layer opening with a downsampling unit; CIFAR / ImageNet32 stem
3x3/s1 without max-pool, ImageNet stem 7x7/s2 + max-pool 3x3/s2.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _lib as L

BASIC = {"revnet18": [2, 2, 2, 2], "revnet34": [3, 4, 6, 3]}
BOTTLENECK = {"revnet50": [3, 4, 6, 3]}
WIDTHS = [64, 128, 256, 512]


@dataclass
class Unit:
    kind: int
    dst: int = 0
    layers: list = field(default_factory=list)   # [(cin, cout, k, s)]
    proj: list = field(default_factory=list)     # DS: [(cin, cout, 1, s)] x 2
    maxpool: int = 0
    classes: int = 0

    def to_c(self) -> L.PetraUnit:
        u = L.PetraUnit()
        u.kind, u.dst_half, u.n_layers = self.kind, self.dst, len(self.layers)
        for i, (ci, co, k, s) in enumerate(self.layers):
            u.layer[i] = L.PetraConv(ci, co, k, s)
        for i, (ci, co, k, s) in enumerate(self.proj):
            u.proj[i] = L.PetraConv(ci, co, k, s)
        u.maxpool, u.classes = self.maxpool, self.classes
        return u


def revnet(name: str, image_size: int = 32, classes: int = 10):
    big = image_size >= 128
    units = [Unit(L.UNIT_STEM, layers=[(3, 128, 7 if big else 3, 2 if big else 1)], maxpool=int(big))]
    if name in BASIC:
        cp = 64
        for li, nb in enumerate(BASIC[name]):
            c = WIDTHS[li]
            for b in range(nb):
                if b == 0 and li > 0:
                    units.append(Unit(L.UNIT_DS, 0, [(cp, c, 3, 2)], [(cp, c, 1, 2), (cp, c, 1, 2)]))
                else:
                    units.append(Unit(L.UNIT_REV, 0, [(c, c, 3, 1)]))
                units.append(Unit(L.UNIT_REV, 1, [(c, c, 3, 1)]))
            cp = c
    elif name in BOTTLENECK:
        cp = 64
        for li, nb in enumerate(BOTTLENECK[name]):
            mid = WIDTHS[li]
            c, s = 4 * mid, (1 if li == 0 else 2)
            units.append(Unit(L.UNIT_DS, 0, [(cp, mid, 1, 1), (mid, mid, 3, s), (mid, c, 1, 1)],
                              [(cp, c, 1, s), (cp, c, 1, s)]))
            for b in range(1, nb):
                units.append(Unit(L.UNIT_REV, (b - 1) % 2, [(c, mid, 1, 1), (mid, mid, 3, 1), (mid, c, 1, 1)]))
            cp = c
    else:
        raise ValueError(f"unknown model {name}")
    units.append(Unit(L.UNIT_TAIL, classes=classes))
    return units


def mlp(d: int = 64, classes: int = 10):
    """Config 1: F/G units of Linear(d/2 -> d/2)-BN-ReLU on [B, d/2, 1, 1] halves."""
    h = d // 2
    rv = lambda dst: Unit(L.UNIT_REV, dst, [(h, h, 1, 1)])
    return [rv(0), rv(1), rv(0), rv(1), Unit(L.UNIT_TAIL, classes=classes)]


def _out(n, k, s):
    return (n + 2 * ((k - 1) // 2) - k) // s + 1


def shapes(units, batch, h, w, c):
    """Per-unit input shapes (B, H, W, C_half-or-image) and the final shape."""
    cur = (batch, h, w, c)
    ins = []
    for u in units:
        ins.append(cur)
        B, H, W, Cc = cur
        if u.kind == L.UNIT_STEM:
            ci, co, k, s = u.layers[0]
            H, W = _out(H, k, s), _out(W, k, s)
            if u.maxpool:
                H, W = (H - 1) // 2 + 1, (W - 1) // 2 + 1
            cur = (B, H, W, co // 2)
        elif u.kind == L.UNIT_DS:
            ci, co, k, s = u.proj[0]
            cur = (B, _out(H, 1, s), _out(W, 1, s), co)
    return ins, cur


def conv_macs(units, batch, h, w, c):
    """Forward multiply-accumulates per unit (conv layers; FC for the tail)."""
    ins, _ = shapes(units, batch, h, w, c)
    out = []
    for u, (B, H, W, Cc) in zip(units, ins):
        tot = 0

        def chain(layers, H, W):
            t = 0
            for ci, co, k, s in layers:
                H, W = _out(H, k, s), _out(W, k, s)
                t += B * H * W * co * ci * k * k
            return t
        if u.kind in (L.UNIT_REV, L.UNIT_DS, L.UNIT_STEM):
            tot += chain(u.layers, H, W)
        if u.kind == L.UNIT_DS:
            for p in u.proj:
                tot += chain([p], H, W)
        if u.kind == L.UNIT_TAIL:
            tot += B * 2 * Cc * u.classes
        out.append(tot)
    return out


def partition(units, J, batch=64, h=32, w=32, c=3):
    """Contiguous FLOP-balanced grouping of units into J stages (reading c14):
    minimises the largest stage (binary search on the bottleneck)."""
    cost = conv_macs(units, batch, h, w, c)
    n = len(units)
    if J > n:
        raise ValueError(f"J={J} > {n} units")

    def fits(cap):
        counts, cur, k = [], 0, 0
        for i, x in enumerate(cost):
            if k and cur + x > cap:
                counts.append(k)
                cur, k = 0, 0
            cur += x
            k += 1
        counts.append(k)
        return counts if len(counts) <= J else None

    lo, hi = max(cost), sum(cost)
    while lo < hi:
        mid = (lo + hi) // 2
        if fits(mid):
            hi = mid
        else:
            lo = mid + 1
    counts = fits(lo)
    while len(counts) < J:             # split the largest multi-unit stage
        i = max((i for i in range(len(counts)) if counts[i] > 1), key=lambda i: counts[i])
        counts[i:i + 1] = [counts[i] - counts[i] // 2, counts[i] // 2]
    return counts


# ---- cost model of a unit's tick (comm-aware partitioner)
# Measured on B200 (profiles/r01, serialised replay): tensor-core convolutions run
# at ~0.27 of the bf16 peak inside a tick, the streaming BN / coupling passes at
# ~0.6 of HBM; a peer copy over NVLink 5 at 770 GB/s per direction (B200_PROFILING.md).
TC_FLOPS = 0.27 * 1.37e15
HBM_BPS = 0.6 * 6.46e12
LINK_BPS = 7.7e11


def unit_cost(units, batch, h, w, c):
    """Modelled device seconds of one tick of each unit (forward + reconstruction +
    VJP = 4x the forward conv FLOPs for reversible units, Table 1; the
    same count for non-reversible units, which recompute from their buffer) plus its
    streaming bytes: per half-coupling the forward reads src/dst and writes dst
    (3 N fp32), the backward reads dst', src, d_dst, d_src and writes dst, d_src
    (6 N), and every conv output is written and read in bf16 in the forward, the
    recomputation and twice in the BN backward."""
    macs = conv_macs(units, batch, h, w, c)
    ins, _ = shapes(units, batch, h, w, c)
    out = []
    for u, m, (B, H, W, Cc) in zip(units, macs, ins):
        flops = 4 * 2.0 * m
        by = 0.0
        if u.kind in (L.UNIT_REV, L.UNIT_DS):
            n = B * H * W * Cc
            by += 9 * 4.0 * n
            HH, WW = H, W
            for ci, co, k, s in u.layers:
                HH, WW = _out(HH, k, s), _out(WW, k, s)
                by += 4 * 2.0 * B * HH * WW * co
        elif u.kind == L.UNIT_STEM:
            ci, co, k, s = u.layers[0]
            by += 4 * 2.0 * B * _out(H, k, s) * _out(W, k, s) * co + 3 * 4.0 * B * H * W * Cc
        out.append(flops / TC_FLOPS + by / HBM_BPS)
    return out


def boundary_bytes(units, batch, h, w, c):
    """Bytes crossing the cut in front of unit i per tick: the forward message
    (2 fp32 halves) plus the backward message (x~ and delta: 4 halves)."""
    ins, _ = shapes(units, batch, h, w, c)
    return [6 * 4.0 * B * H * W * Cc for (B, H, W, Cc) in ins]


def partition_comm(units, J, world, batch=64, h=32, w=32, c=3):
    """Contiguous grouping of units into J stages on `world` GPUs (J/world
    consecutive stages per GPU, contiguous_stage_ranks) minimising the slowest GPU:
    max over GPUs of (its stages' modelled compute + the bytes of its cross-GPU cuts
    / link).  Exact by dynamic programming over cut positions (units <= ~20)."""
    cost = unit_cost(units, batch, h, w, c)
    bnd = boundary_bytes(units, batch, h, w, c)
    n = len(units)
    if J > n:
        raise ValueError(f"J={J} > {n} units")
    base, rem = divmod(J, world)
    per_gpu = [base + (1 if r < rem else 0) for r in range(world)]
    pre = [0.0]
    for x in cost:
        pre.append(pre[-1] + x)
    import functools

    @functools.lru_cache(maxsize=None)
    def best(i, g):
        """(bottleneck, counts) for units i.. on GPUs g.. ; GPU g takes per_gpu[g] stages."""
        if g == world:
            return (0.0, ()) if i == n else (float("inf"), ())
        k = per_gpu[g]
        rest = sum(per_gpu[g + 1:])
        res = (float("inf"), ())
        for j in range(i + k, n - rest + 1):   # GPU g gets units i..j-1 (>= k of them)
            comm = (bnd[i] if i > 0 else 0.0) + (bnd[j] if j < n else 0.0)
            t = pre[j] - pre[i] + comm / LINK_BPS
            tail, cnts = best(j, g + 1)
            b = max(t, tail)
            if b < res[0]:
                res = (b, (j - i,) + cnts)
        return res

    _, per = best(0, 0)
    # split each GPU's units into its stages, balancing modelled cost inside the GPU
    counts, i = [], 0
    for g, m in enumerate(per):
        sub = units[i:i + m]
        if per_gpu[g] == 1:
            counts.append(m)
        else:
            cs = cost[i:i + m]
            counts += _balance(cs, per_gpu[g])
        i += m
    return counts


def _balance(cost, k):
    """Contiguous split of a cost list into k non-empty groups minimising the maximum."""
    n = len(cost)
    import functools

    @functools.lru_cache(maxsize=None)
    def f(i, k):
        if k == 1:
            return (sum(cost[i:]), (n - i,))
        res = (float("inf"), ())
        for j in range(i + 1, n - k + 2):
            tail = f(j, k - 1)
            b = max(sum(cost[i:j]), tail[0])
            if b < res[0]:
                res = (b, (j - i,) + tail[1])
        return res
    return list(f(0, k)[1])


@dataclass
class StageSpec:
    units: list
    batch: int
    in_shape: tuple   # (H, W, C)
    precision: int = L.FP32
    momentum: float = 0.9
    weight_decay: float = 5e-4
    bn_momentum: float = 0.1
    bn_eps: float = 1e-5
    fifo_capacity: int = 1
    accumulation_k: int = 1   # Alg. 1 lines 19-23
    compare_buffers: int = 0  # Table 3 comparison modes (petra.h PETRA_CMP_INPUTS / PETRA_CMP_STASH)

    def to_c(self):
        arr = (L.PetraUnit * len(self.units))(*[u.to_c() for u in self.units])
        d = L.PetraStageDesc()
        d.n_units, d.units = len(self.units), C.cast(arr, C.POINTER(L.PetraUnit))
        d.batch = self.batch
        d.in_h, d.in_w, d.in_c = self.in_shape
        d.precision, d.momentum, d.weight_decay = self.precision, self.momentum, self.weight_decay
        d.bn_momentum, d.bn_eps, d.nesterov, d.accumulation_k = self.bn_momentum, self.bn_eps, 1, self.accumulation_k
        d.fifo_capacity = self.fifo_capacity
        d.compare_buffers = self.compare_buffers
        return d, arr   # keep arr alive with d


def stage_specs(units, counts, batch, image_hwc, precision=L.FP32, weight_decay=5e-4, accumulation_k=1):
    ins, _ = shapes(units, batch, *image_hwc)
    out, i = [], 0
    J = len(counts)
    for j, n in enumerate(counts, 1):
        B, H, W, Cc = ins[i]
        out.append(StageSpec(units[i:i + n], batch, (H, W, Cc), precision, weight_decay=weight_decay,
                             fifo_capacity=2 * (J - j) + 1, accumulation_k=accumulation_k))
        i += n
    return out
