"""PETRA fp64 CPU oracle -- units (reversible half-coupling, downsampling, stem, tail).

TEST INFRASTRUCTURE, NOT PRODUCT CODE (see oracle/primitives.py header).

A stage is an ordered list of units acting on a list of activation tensors.
Between units the activation is the two-stream pair [x1, x2] (PAPER.md:50-51,
"split equally into {x_j^1, x_j^2} along the channel dimension"); the stem
consumes the single image tensor [x0].

Reversible unit = additive half-coupling  dst <- dst + Phi(src)  (reading c1):
the north_star block  y1 = x1 + F(x2),  y2 = x2 + G(y1)  is the unit pair
[dst=0, Phi=F] then [dst=1, Phi=G]; its inverse subtracts in reverse order
("subtracting the output of F~_j rather than adding it"; Eq. 4).
Phi is a chain of conv(no bias)-BN-ReLU layers (reading c2).
"""
from __future__ import annotations

import numpy as np

from . import primitives as P


class ConvBN:
    """conv(no bias) -> BN(train) [-> ReLU].  Parameters: w (decayed), gamma, beta
    (not decayed, "we do not apply weight decay on the batch norm
    learnable parameters").  Running stats are buffers, not parameters."""

    def __init__(self, cin, cout, k, stride=1, relu=True):
        self.cin, self.cout, self.k, self.stride = cin, cout, k, stride
        self.pad = (k - 1) // 2
        self.act = relu
        self.w = np.zeros((cout, cin, k, k))
        self.gamma = np.ones(cout)
        self.beta = np.zeros(cout)
        self.rmean = np.zeros(cout)
        self.rvar = np.ones(cout)

    def params(self):
        return [("w", self.w, True), ("gamma", self.gamma, False), ("beta", self.beta, False)]

    def buffers(self):
        return [("rmean", self.rmean), ("rvar", self.rvar)]

    def forward(self, x, update_stats=False):
        z = P.conv2d(x, self.w, self.stride, self.pad)
        y, bc = P.bn_train_forward(z, self.gamma, self.beta)
        if update_stats:
            P.bn_running_update(self.rmean, self.rvar, bc)
        mask = None
        if self.act:
            y, mask = P.relu(y)
        return P.stored(y), (x, bc, mask)

    def vjp(self, cache, dout, need_dx=True):
        x, bc, mask = cache
        g = dout * mask if self.act else dout
        dz, dgamma, dbeta = P.bn_train_vjp(bc, self.gamma, g)
        dx, dw = P.conv2d_vjp(x, self.w, self.stride, self.pad, P.stored(dz), need_dx)
        return dx, [dw, dgamma, dbeta]

    def flops_fwd(self, x_shape):
        B, C, H, W = x_shape
        Ho = P.conv_out_size(H, self.k, self.stride, self.pad)
        Wo = P.conv_out_size(W, self.k, self.stride, self.pad)
        return 2 * B * Ho * Wo * self.cout * self.cin * self.k * self.k


class Branch:
    """Phi = chain of ConvBN layers (1 layer: RevNet-18/34 basic; 3 layers:
    RevNet-50 bottleneck 1x1 -> 3x3 -> 1x1, reading c3)."""

    def __init__(self, layers):
        self.layers = list(layers)

    def params(self):
        return [p for l in self.layers for p in l.params()]

    def buffers(self):
        return [b for l in self.layers for b in l.buffers()]

    def forward(self, x, update_stats=False):
        caches = []
        for l in self.layers:
            x, c = l.forward(x, update_stats)
            caches.append(c)
        return x, caches

    def vjp(self, caches, dout, need_dx=True):
        grads = []
        for i in range(len(self.layers) - 1, -1, -1):
            dout, g = self.layers[i].vjp(caches[i], dout, need_dx or i > 0)
            grads = g + grads
        return dout, grads

    def flops_fwd(self, x_shape):
        total, shape = 0, x_shape
        for l in self.layers:
            total += l.flops_fwd(shape)
            B, C, H, W = shape
            shape = (B, l.cout, P.conv_out_size(H, l.k, l.stride, l.pad),
                     P.conv_out_size(W, l.k, l.stride, l.pad))
        return total


class RevUnit:
    """Additive half-coupling  x[dst] <- x[dst] + Phi(x[src])  (reversible).

    forward        : PAPER.md:131  x_j^{t+1} = F_j(x_{j-1}^t, theta^t)
    reconstruct    : PAPER.md:132  x~_{j-1} = F_j^{-1}(x~_j, theta^t) -- subtract
                     Phi evaluated with the CURRENT parameters, keep the graph,
                     update BN running stats
    vjp            : PAPER.md:133-134 delta and Delta at (x~, theta^t)
    """
    reversible = True

    def __init__(self, dst, phi: Branch):
        assert dst in (0, 1)
        self.dst, self.src, self.phi = dst, 1 - dst, phi

    def params(self):
        return self.phi.params()

    def buffers(self):
        return self.phi.buffers()

    def forward(self, xs, update_stats=False):
        ys, _ = self.forward_graph(xs, update_stats)
        return ys

    def forward_graph(self, xs, update_stats=False):
        out, caches = self.phi.forward(xs[self.src], update_stats)
        ys = list(xs)
        ys[self.dst] = P.stored(xs[self.dst] + out)
        return ys, caches

    def reconstruct(self, ys):
        out, caches = self.phi.forward(ys[self.src], update_stats=True)
        xs = list(ys)
        xs[self.dst] = P.stored(ys[self.dst] - out)
        return xs, caches

    def vjp(self, caches, ds):
        dsrc, grads = self.phi.vjp(caches, ds[self.dst])
        out = list(ds)
        out[self.src] = P.stored(ds[self.src] + dsrc)   # delta of dst passes through unchanged
        return out, grads

    def flops_fwd(self, shapes):
        return self.phi.flops_fwd(shapes[self.src])

    def out_shapes(self, shapes):
        return list(shapes)


class DSUnit:
    """Non-reversible downsampling unit ("only a few stages which do
    not preserve feature dimensionality are not reversible"; reading c3):

        y[dst] = P_a(x[dst]) + Phi_s(x[src]),   y[src] = P_b(x[src])

    Phi_s: conv-BN-ReLU branch whose 3x3 has stride s; P_a, P_b: conv1x1/s + BN.
    Handled by buffering the input and recomputing."""
    reversible = False

    def __init__(self, dst, phi: Branch, pa: ConvBN, pb: ConvBN):
        self.dst, self.src = dst, 1 - dst
        self.phi, self.pa, self.pb = phi, pa, pb

    def params(self):
        return self.phi.params() + self.pa.params() + self.pb.params()

    def buffers(self):
        return self.phi.buffers() + self.pa.buffers() + self.pb.buffers()

    def forward_graph(self, xs, update_stats=False):
        phi_out, c_phi = self.phi.forward(xs[self.src], update_stats)
        pa_out, c_pa = self.pa.forward(xs[self.dst], update_stats)
        pb_out, c_pb = self.pb.forward(xs[self.src], update_stats)
        ys = [None, None]
        ys[self.dst] = P.stored(pa_out + phi_out)
        ys[self.src] = pb_out
        return ys, (c_phi, c_pa, c_pb)

    def vjp(self, graph, ds, need_dx=True):
        c_phi, c_pa, c_pb = graph
        d_src_phi, g_phi = self.phi.vjp(c_phi, ds[self.dst], need_dx)
        d_dst, g_pa = self.pa.vjp(c_pa, ds[self.dst], need_dx)
        d_src_pb, g_pb = self.pb.vjp(c_pb, ds[self.src], need_dx)
        out = [None, None]
        if need_dx:
            out[self.dst] = d_dst
            out[self.src] = P.stored(d_src_phi + d_src_pb)
        return out, g_phi + g_pa + g_pb

    def flops_fwd(self, shapes):
        return (self.phi.flops_fwd(shapes[self.src]) + self.pa.flops_fwd(shapes[self.dst])
                + self.pb.flops_fwd(shapes[self.src]))


class StemUnit:
    """Input layer: conv(k, stride) -> BN -> ReLU [-> max-pool 3x3/s2], output
    channels split into the two streams (first half -> x1).  PAPER.md:259: CIFAR
    uses a 3x3 conv without max-pool; ImageNet the 7x7/s2 conv with max-pool.
    Non-reversible: its input x0 is buffered."""
    reversible = False

    def __init__(self, cin, cout, k, stride, maxpool):
        self.layer = ConvBN(cin, cout, k, stride, relu=True)
        self.maxpool = maxpool

    def params(self):
        return self.layer.params()

    def buffers(self):
        return self.layer.buffers()

    def forward_graph(self, xs, update_stats=False):
        (x0,) = xs
        a, c = self.layer.forward(x0, update_stats)
        mp = None
        if self.maxpool:
            a_shape = a.shape
            a, arg = P.maxpool3x3s2(a)
            mp = (a_shape, arg)
        h = a.shape[1] // 2
        return [a[:, :h].copy(), a[:, h:].copy()], (c, mp)

    def vjp(self, graph, ds, need_dx=False):
        c, mp = graph
        d = np.concatenate(ds, axis=1)
        if mp is not None:
            d = P.maxpool3x3s2_vjp(mp[0], mp[1], d)
        dx, g = self.layer.vjp(c, d, need_dx)
        return [dx], g

    def flops_fwd(self, shapes):
        return self.layer.flops_fwd(shapes[0])


class TailUnit:
    """Final stage head: global average pool of concat(x1, x2), Linear(2C ->
    classes) with bias, batch-mean softmax cross-entropy (
    readings c7, c18).  Bias is not decayed."""
    reversible = False
    is_tail = True

    def __init__(self, cin, classes):
        self.cin, self.classes = cin, classes
        self.w = np.zeros((classes, cin))
        self.b = np.zeros(classes)

    def params(self):
        return [("w", self.w, True), ("b", self.b, False)]

    def buffers(self):
        return []

    def loss_graph(self, xs, labels):
        x = np.concatenate(xs, axis=1)
        feat = x.mean(axis=(2, 3))
        logits = P.linear(feat, self.w, self.b)
        loss, dlogits = P.softmax_cross_entropy(logits, labels)
        return loss, (x.shape, feat, dlogits, xs[0].shape[1])

    def vjp(self, graph):
        x_shape, feat, dlogits, c1 = graph
        dw = dlogits.T @ feat
        db = dlogits.sum(axis=0)
        dfeat = dlogits @ self.w
        B, C, H, W = x_shape
        dx = np.broadcast_to((dfeat / (H * W))[:, :, None, None], x_shape).copy()
        return [dx[:, :c1].copy(), dx[:, c1:].copy()], [dw, db]

    def flops_fwd(self, shapes):
        B = shapes[0][0]
        return 2 * B * self.cin * self.classes
