"""Pins of the oracle's units (coupling forward / inverse / VJP, DS, stem, tail)."""
import numpy as np
import pytest

import synth
from oracle import engine as E
from oracle import models as M
from oracle.units import Branch, ConvBN, DSUnit, RevUnit, StemUnit, TailUnit
from tests.torch_ref import TorchNet


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


class ScalePhi:
    """Phi(u) = s*u, a parameter-free branch for the worked example."""

    def __init__(self, s):
        self.s = s

    def params(self):
        return []

    def buffers(self):
        return []

    def forward(self, x, update_stats=False):
        return self.s * x, None

    def vjp(self, caches, d, need_dx=True):
        return self.s * d, []


def test_coupling_worked_example(golden):
    g = golden("coupling_scalar.json")
    F = RevUnit(0, ScalePhi(g["F_scale"]))
    G = RevUnit(1, ScalePhi(g["G_scale"]))
    xs = [np.array([g["x"][0]]), np.array([g["x"][1]])]
    ys = G.forward(F.forward(xs))
    assert [ys[0][0], ys[1][0]] == g["y"]
    # inverse: undo G then F
    r, cg = G.reconstruct(ys)
    r, cf = F.reconstruct(r)
    assert [r[0][0], r[1][0]] == g["x"]
    # VJP: G's vjp first, then F's
    ds = [np.array([g["dy"][0]]), np.array([g["dy"][1]])]
    ds, _ = G.vjp(cg, ds)
    ds, _ = F.vjp(cf, ds)
    assert [ds[0][0], ds[1][0]] == g["dx"]


def rand_unit_params(units, seed):
    """Random theta including non-trivial gamma/beta (so BN is not the identity)."""
    M.init_params(units, seed)
    i = 0
    for u in units:
        for name, p, _ in u.params():
            if name == "gamma":
                p[...] = 1.0 + 0.3 * synth.normal(p.shape, seed, 100, i)
            elif name in ("beta", "b"):
                p[...] = 0.2 * synth.normal(p.shape, seed, 101, i)
            i += 1
    return units


def basic_unit(c, dst):
    return RevUnit(dst, Branch([ConvBN(c, c, 3, 1)]))


def bottleneck_unit(c, mid, dst):
    return RevUnit(dst, Branch([ConvBN(c, mid, 1, 1), ConvBN(mid, mid, 3, 1), ConvBN(mid, c, 1, 1)]))


def test_frozen_theta_inversion_100_draws():
    """PAPER.md:89-101 Eq. 4: at fixed theta the reconstruction is exact
    (||.||_inf < 1e-11 in f64 over >= 100 random draws)."""
    worst = 0.0
    for d in range(100):
        if d % 2 == 0:
            units = [basic_unit(4, 0), basic_unit(4, 1)]
        else:
            units = [bottleneck_unit(8, 2, 0), bottleneck_unit(8, 2, 1)]
        rand_unit_params(units, 1000 + d)
        c = 4 if d % 2 == 0 else 8
        xs = [synth.normal((3, c, 4, 4), d, 1), synth.normal((3, c, 4, 4), d, 2)]
        ys = xs
        for u in units:
            ys = u.forward(ys)
        r = ys
        for u in reversed(units):
            r, _ = u.reconstruct(r)
        worst = max(worst, max(np.max(np.abs(a - b)) for a, b in zip(r, xs)))
    assert worst < 1e-11, worst


def test_inversion_error_is_first_order_in_theta_change():
    """perturbing theta by eps before inversion gives error O(eps):
    ratio err(eps)/err(eps/2) in [1.5, 2.5] (the 'approximate inversion',
    PAPER.md:139)."""
    units = rand_unit_params([basic_unit(4, 0), basic_unit(4, 1)], 7)
    xs = [synth.normal((4, 4, 5, 5), 3, 1), synth.normal((4, 4, 5, 5), 3, 2)]
    ys = units[1].forward(units[0].forward(xs))
    dirs = [synth.normal(p.shape, 8, i) for i, (_, p, _) in enumerate(units[0].params() + units[1].params())]

    def err(eps):
        saved = [p.copy() for (_, p, _) in units[0].params() + units[1].params()]
        for (_, p, _), dd in zip(units[0].params() + units[1].params(), dirs):
            p += eps * dd
        r, _ = units[1].reconstruct(ys)
        r, _ = units[0].reconstruct(r)
        for (_, p, _), s in zip(units[0].params() + units[1].params(), saved):
            p[...] = s
        return np.sqrt(sum(np.sum((a - b) ** 2) for a, b in zip(r, xs)))

    ratio = err(1e-4) / err(0.5e-4)
    assert 1.5 <= ratio <= 2.5, ratio


def test_zero_branch_is_identity():
    """F~ == 0 (gamma=beta=0 makes Phi = ReLU(0) = 0): the unit
    is the identity, delta passes through, all parameter gradients of W vanish."""
    u = basic_unit(3, 0)
    M.init_params([u], 2)
    u.phi.layers[0].gamma[...] = 0.0
    xs = [synth.normal((2, 3, 4, 4), 1), synth.normal((2, 3, 4, 4), 2)]
    ys = u.forward(xs)
    assert all(np.array_equal(a, b) for a, b in zip(ys, xs))
    r, g = u.reconstruct(ys)
    ds = [synth.normal((2, 3, 4, 4), 3), synth.normal((2, 3, 4, 4), 4)]
    out, grads = u.vjp(g, ds)
    assert all(np.array_equal(a, b) for a, b in zip(out, ds))
    assert np.all(grads[0] == 0.0)


def test_fused_backward_equals_naive_path():
    """PAPER.md:307 / SPEC.md:267: reconstruct-with-graph + VJP equals
    inverse, then a fresh forward recording, then VJP -- bitwise in f64."""
    units = rand_unit_params([bottleneck_unit(8, 4, 0), bottleneck_unit(8, 4, 1)], 11)
    xs = [synth.normal((2, 8, 4, 4), 5, 1), synth.normal((2, 8, 4, 4), 5, 2)]
    ys = units[1].forward(units[0].forward(xs))
    ds0 = [synth.normal((2, 8, 4, 4), 6, 1), synth.normal((2, 8, 4, 4), 6, 2)]
    # fused
    r, g1 = units[1].reconstruct(ys)
    d, gr1 = units[1].vjp(g1, ds0)
    r, g0 = units[0].reconstruct(r)
    d, gr0 = units[0].vjp(g0, d)
    # naive
    u1x = list(ys)
    u1x[1] = ys[1] - units[1].phi.forward(ys[0])[0]
    _, g1n = units[1].forward_graph(u1x)
    dn, gr1n = units[1].vjp(g1n, ds0)
    u0x = list(u1x)
    u0x[0] = u1x[0] - units[0].phi.forward(u1x[1])[0]
    _, g0n = units[0].forward_graph(u0x)
    dn, gr0n = units[0].vjp(g0n, dn)
    assert all(np.array_equal(a, b) for a, b in zip(r, u0x))
    assert all(np.array_equal(a, b) for a, b in zip(d, dn))
    assert all(np.array_equal(a, b) for a, b in zip(gr0 + gr1, gr0n + gr1n))


def tiny_net(maxpool):
    """Every unit kind in one small net: stem(+max-pool), basic rev, basic DS,
    bottleneck DS, bottleneck rev, tail."""
    return [
        StemUnit(3, 8, 3, 1 if not maxpool else 2, maxpool),
        basic_unit(4, 0), basic_unit(4, 1),
        DSUnit(0, Branch([ConvBN(4, 6, 3, 2)]), ConvBN(4, 6, 1, 2, relu=False), ConvBN(4, 6, 1, 2, relu=False)),
        basic_unit(6, 1),
        DSUnit(0, Branch([ConvBN(6, 2, 1, 1), ConvBN(2, 2, 3, 2), ConvBN(2, 8, 1, 1)]),
               ConvBN(6, 8, 1, 2, relu=False), ConvBN(6, 8, 1, 2, relu=False)),
        bottleneck_unit(8, 2, 1),
        TailUnit(16, 5),
    ]


@pytest.mark.parametrize("maxpool", [False, True])
def test_backprop_vs_torch_autograd(maxpool):
    """Oracle backprop (hand-written VJPs, Eqs. 2-3) against
    torch.autograd on an independent torch.nn.functional forward, fp64."""
    units = rand_unit_params(tiny_net(maxpool), 21)
    H = 16 if maxpool else 8
    x0 = synth.images((3, 3, H, H), 0, 0)
    lab = synth.labels(3, 5, 0, 0)
    tn = TorchNet(units)
    tloss, tgrads = tn.grads([x0], lab)
    loss, grads = E.backprop_grads(units, [x0], lab)
    assert abs(loss - tloss) < 1e-13 * abs(tloss)
    assert len(grads) == len(tgrads)
    for g, t in zip(grads, tgrads):
        # some BN shifts are annihilated downstream (true gradient ~1e-17): absolute floor
        assert np.linalg.norm(g - t) <= 1e-9 * np.linalg.norm(t) + 1e-13


def test_backprop_finite_difference():
    """FD of the total loss wrt every parameter tensor of a
    composed network, h=1e-5, rel 1e-4 (directional derivatives)."""
    units = rand_unit_params(tiny_net(False), 31)
    x0 = synth.images((4, 3, 8, 8), 0, 1)
    lab = synth.labels(4, 5, 0, 1)
    _, grads = E.backprop_grads(units, [x0], lab)
    params = [p for u in units for (_, p, _) in u.params()]
    for i, (p, g) in enumerate(zip(params, grads)):
        d = synth.normal(p.shape, 40, i)
        an = float(np.sum(g * d))
        errs = []
        # h=1e-5 per SPEC.md:116; h=1e-6 as well because a ReLU kink within h of a
        # pre-activation corrupts one of the two central differences
        for h in (1e-5, 1e-6):
            p += h * d
            lp, _ = E.backprop_grads(units, [x0], lab)
            p -= 2 * h * d
            lm, _ = E.backprop_grads(units, [x0], lab)
            p += h * d
            errs.append(abs((lp - lm) / (2 * h) - an))
        assert min(errs) <= 1e-4 * abs(an) + 1e-9, (i, errs, an)


def test_unit_vjp_linearity():
    """vjp(a d1 + b d2) == a vjp(d1) + b vjp(d2) (1e-12)."""
    u = rand_unit_params([bottleneck_unit(8, 4, 1)], 3)[0]
    xs = [synth.normal((2, 8, 3, 3), 1), synth.normal((2, 8, 3, 3), 2)]
    _, g = u.forward_graph(xs)
    d1 = [synth.normal((2, 8, 3, 3), 3), synth.normal((2, 8, 3, 3), 4)]
    d2 = [synth.normal((2, 8, 3, 3), 5), synth.normal((2, 8, 3, 3), 6)]
    a, b = 0.7, -1.3
    o1, g1 = u.vjp(g, d1)
    o2, g2 = u.vjp(g, d2)
    o3, g3 = u.vjp(g, [a * x + b * y for x, y in zip(d1, d2)])
    for x, y, z in zip(o1 + g1, o2 + g2, o3 + g3):
        assert np.max(np.abs(a * x + b * y - z)) < 1e-12 * max(1.0, np.max(np.abs(z)))
