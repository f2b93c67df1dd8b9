"""Independent fp64 reference built on torch.nn.functional + torch.autograd.

Used only by the oracle pin tests: it re-expresses the network forward with a
different library (F.conv2d, F.batch_norm, F.relu, F.max_pool2d,
F.cross_entropy) and lets autograd produce the backprop gradients, so a
mistake in the oracle's hand-written VJPs (dropped term, wrong sign, transposed
operand) shows up as a mismatch.
"""
import numpy as np
import torch
import torch.nn.functional as TF

from oracle.units import ConvBN, DSUnit, RevUnit, StemUnit, TailUnit


def _t(a):
    return torch.tensor(a, dtype=torch.float64, requires_grad=True)


class TorchNet:
    def __init__(self, units):
        self.units = units
        self.leaves = [[_t(p) for (_, p, _) in u.params()] for u in units]

    def _cbr(self, layer: ConvBN, x, w, g, b):
        z = TF.conv2d(x, w, stride=layer.stride, padding=layer.pad)
        y = TF.batch_norm(z, None, None, g, b, training=True, eps=1e-5)
        return TF.relu(y) if layer.act else y

    def _branch(self, branch, x, leaves):
        for i, l in enumerate(branch.layers):
            x = self._cbr(l, x, *leaves[3 * i:3 * i + 3])
        return x

    def forward(self, xs, labels=None):
        xs = [torch.tensor(x, dtype=torch.float64) for x in xs]
        for u, lv in zip(self.units, self.leaves):
            if isinstance(u, RevUnit):
                ys = list(xs)
                ys[u.dst] = xs[u.dst] + self._branch(u.phi, xs[u.src], lv)
                xs = ys
            elif isinstance(u, DSUnit):
                n = 3 * len(u.phi.layers)
                phi = self._branch(u.phi, xs[u.src], lv[:n])
                pa = self._cbr(u.pa, xs[u.dst], *lv[n:n + 3])
                pb = self._cbr(u.pb, xs[u.src], *lv[n + 3:n + 6])
                ys = [None, None]
                ys[u.dst] = pa + phi
                ys[u.src] = pb
                xs = ys
            elif isinstance(u, StemUnit):
                a = self._cbr(u.layer, xs[0], *lv)
                if u.maxpool:
                    a = TF.max_pool2d(a, 3, 2, 1)
                h = a.shape[1] // 2
                xs = [a[:, :h], a[:, h:]]
            elif isinstance(u, TailUnit):
                feat = torch.cat(xs, 1).mean(dim=(2, 3))
                logits = feat @ lv[0].T + lv[1]
                return TF.cross_entropy(logits, torch.tensor(labels))
        return xs

    def grads(self, xs, labels):
        loss = self.forward(xs, labels)
        flat = [t for lv in self.leaves for t in lv]
        gs = torch.autograd.grad(loss, flat)
        return loss.item(), [g.numpy() for g in gs]
