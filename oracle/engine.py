"""PETRA fp64 CPU oracle -- stage worker (Alg. 1), optimizer, tick engine and the
reference modes (lockstep, monolithic backprop).

TEST INFRASTRUCTURE, NOT PRODUCT CODE (see oracle/primitives.py header).

Tick semantics (PAPER.md:127-137 equation system, readings c8/c12; SURVEY §8(c)
step 7): mailboxes are double-buffered -- a message produced at tick t is
visible at t+1.  At tick t every stage j (1) runs its forward at theta^t on the
message received from j-1 (stage 1 reads micro-batch m=t), (2) runs its
backward at theta^t on the message received from j+1 (the last stage runs its
own forward+loss+backward in the same tick), (3) applies the update giving
theta^{t+1}.  Hence stage j forwards mb m at t_f = m+j-1 and backwards it at
t_b = m+2J-j-1: delay 2(J-j) (Table 1).
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np


# --------------------------------------------------------------------------- optimizer
@dataclass
class OptConfig:
    """SGD with Nesterov momentum 0.9, L2 weight decay folded into
    the gradient and skipped for BN parameters and biases,
    accumulation factor k with averaged gradients."""
    momentum: float = 0.9
    weight_decay: float = 5e-4
    nesterov: bool = True
    k: int = 1


def sgd_step(theta, v, grad, lr, cfg: OptConfig, decay: bool):
    """Reading c11 (PyTorch SGD, dampening 0):  g = Delta + lambda*theta;
    v <- mu*v + g;  theta <- theta - lr*(g + mu*v)  (Nesterov) or theta - lr*v."""
    g = grad + cfg.weight_decay * theta if decay else grad.copy()
    v *= cfg.momentum
    v += g
    if cfg.nesterov:
        theta -= lr * (g + cfg.momentum * v)
    else:
        theta -= lr * v


def scaled_base_lr(k: int, micro_batch: int = 64) -> float:
    """lr = 0.1 * 64k / 256."""
    return 0.1 * micro_batch * k / 256.0


# --------------------------------------------------------------------------- messages
@dataclass
class Fwd:
    mb: int
    xs: list
    labels: np.ndarray


@dataclass
class Bwd:
    mb: int
    xs: list      # reconstructed activation x~
    ds: list      # gradient delta


# --------------------------------------------------------------------------- stage
class Stage:
    """One PETRA worker (Alg. 1).  Holds a single parameter
    version ("avoiding weight stashing"), optimizer slots, the
    accumulator Delta_j, the local step counter t, and one input FIFO per
    non-reversible unit (reading c5: the INPUT is buffered)."""

    def __init__(self, units, opt: OptConfig, j: int = 1, J: int = 1):
        self.units = list(units)
        self.opt = opt
        self.j, self.J = j, J
        self.is_last = getattr(self.units[-1], "is_tail", False)
        self.fifo = {i: deque() for i, u in enumerate(self.units) if not u.reversible}
        self.fifo_peak = {i: 0 for i in self.fifo}
        self.v = [np.zeros_like(p) for (_, p, _) in self.params()]
        self.acc = [np.zeros_like(p) for (_, p, _) in self.params()]
        self.t = 1               # reading c12: t starts at 1, counts backwards
        self.version = 0         # number of optimizer updates applied so far
        self.n_fwd = self.n_bwd = 0
        self.last_grads = None   # unscaled Delta of the last backward (for tests)

    def params(self):
        return [p for u in self.units for p in u.params()]

    def buffers(self):
        return [b for u in self.units for b in u.buffers()]

    # ---- forward branch (Alg. 1 lines 3-10)
    def forward(self, msg: Fwd) -> Fwd:
        xs = list(msg.xs)
        for i, u in enumerate(self.units):
            if u.reversible:
                xs = u.forward(xs, update_stats=False)      # PAPER.md:259 no stat update
            else:
                self.fifo[i].append((msg.mb, [x.copy() for x in xs]))   # Buffer_j <- input (c5)
                self.fifo_peak[i] = max(self.fifo_peak[i], len(self.fifo[i]))
                xs, _ = u.forward_graph(xs, update_stats=False)
        self.n_fwd += 1
        return Fwd(msg.mb, xs, msg.labels)

    # ---- backward branch (Alg. 1 lines 11-24)
    def backward(self, msg: Bwd, need_input_grad: bool = True) -> Bwd:
        xs, ds = list(msg.xs), list(msg.ds)
        grads = []
        for i in range(len(self.units) - 1, -1, -1):
            u = self.units[i]
            if u.reversible:
                xs, graph = u.reconstruct(xs)               # line 14 + keep graph
                ds, g = u.vjp(graph, ds)                    # lines 18-19
            else:
                if not self.fifo[i]:
                    raise RuntimeError("non-reversible backward with empty buffer (schedule bug)")
                mb, xin = self.fifo[i].popleft()            # line 16
                if mb != msg.mb:
                    raise RuntimeError(f"FIFO order: head mb {mb} != backward mb {msg.mb}")
                _, graph = u.forward_graph(xin, update_stats=True)   # line 17: recompute graph
                first = (i == 0 and self.j == 1)
                ds, g = u.vjp(graph, ds, need_dx=(need_input_grad or not first))
                xs = xin                                     # exact buffered input (c6)
            grads = g + grads
        self._accumulate_and_update(grads, msg)
        self.n_bwd += 1
        return Bwd(msg.mb, xs, ds)

    # ---- final stage (Alg. 1 lines 26-35): forward, loss, backprop, update
    def tail_step(self, msg: Fwd):
        xs = list(msg.xs)
        graphs = []
        for u in self.units[:-1]:
            if u.reversible:
                xs, graph = u.forward_graph(xs, update_stats=True)   # reading c10
            else:
                xs, graph = u.forward_graph(xs, update_stats=True)
            graphs.append(graph)
        loss, tgraph = self.units[-1].loss_graph(xs, msg.labels)
        ds, grads = self.units[-1].vjp(tgraph)
        for i in range(len(self.units) - 2, -1, -1):
            u = self.units[i]
            if u.reversible:
                ds, g = u.vjp(graphs[i], ds)
            else:
                first = (i == 0 and self.j == 1)
                ds, g = u.vjp(graphs[i], ds, need_dx=not first)
            grads = g + grads
        self._accumulate_and_update(grads, msg)
        self.n_fwd += 1
        self.n_bwd += 1
        # reading c7: the tail sends back the RECEIVED input x_{J-1} and delta_J
        return loss, Bwd(msg.mb, list(msg.xs), ds)

    def _accumulate_and_update(self, grads, msg):
        ps = self.params()
        assert len(grads) == len(ps)
        self.last_grads = [g.copy() for g in grads]
        k = self.opt.k
        for a, g in zip(self.acc, grads):
            a += g / k                                       # line 19
        if self.t % k == 0:                                  # line 20
            for (_, p, decay), v, a in zip(ps, self.v, self.acc):
                sgd_step(p, v, a, self.lr, self.opt, decay)  # line 21
                a[...] = 0.0                                 # line 22
            self.version += 1
        self.t += 1                                          # line 23

    lr = 0.0   # set by the engine before each tick (a per-tick scalar input)


# --------------------------------------------------------------------------- engines
@dataclass
class TickReport:
    """Integer bookkeeping per tick; compared bit-exactly."""
    tick: int
    fwd_mb: list = field(default_factory=list)     # per stage, -1 = idle
    bwd_mb: list = field(default_factory=list)
    version: list = field(default_factory=list)    # param version used this tick
    fifo_depth: list = field(default_factory=list) # summed over the stage's FIFOs, after the tick
    loss: float = float("nan")


def run_petra(stages, batch_fn, n_mb: int, lr=0.0, drain: bool = True, record_grads=False,
              n_ticks: int | None = None):
    """Decoupled PETRA schedule over ``n_mb`` micro-batches.

    batch_fn(m) -> (xs0, labels): stage-1 input message for micro-batch m.
    Returns (reports, losses{mb: loss}, grads{(j, mb): [Delta]}).
    """
    J = len(stages)
    for j, s in enumerate(stages, 1):
        s.j, s.J = j, J
    fwd_box = [None] * (J + 2)   # fwd_box[j]: message for stage j (from j-1)
    bwd_box = [None] * (J + 2)   # bwd_box[j]: message for stage j (from j+1)
    total = n_ticks if n_ticks is not None else (n_mb + 2 * J - 2 if drain else n_mb)
    reports, losses, grads = [], {}, {}
    for t in range(total):
        lr_t = lr(t) if callable(lr) else lr
        new_fwd = [None] * (J + 2)
        new_bwd = [None] * (J + 2)
        rep = TickReport(t)
        for j, s in enumerate(stages, 1):
            s.lr = lr_t
            rep.version.append(s.version)
            fin = None
            if j == 1:
                if t < n_mb:
                    xs0, lab = batch_fn(t)
                    fin = Fwd(t, list(xs0), lab)
            else:
                fin = fwd_box[j]
            fmb = bmb = -1
            if j < J:
                if fin is not None:
                    new_fwd[j + 1] = s.forward(fin)
                    fmb = fin.mb
                bin_ = bwd_box[j]
                if bin_ is not None:
                    out = s.backward(bin_)
                    bmb = bin_.mb
                    if record_grads:
                        grads[(j, bin_.mb)] = s.last_grads
                    if j > 1:
                        new_bwd[j - 1] = out
            else:
                if fin is not None:
                    loss, out = s.tail_step(fin)
                    fmb = bmb = fin.mb
                    losses[fin.mb] = loss
                    rep.loss = loss
                    if record_grads:
                        grads[(j, fin.mb)] = s.last_grads
                    if j > 1:
                        new_bwd[j - 1] = out
            rep.fwd_mb.append(fmb)
            rep.bwd_mb.append(bmb)
            rep.fifo_depth.append(sum(len(q) for q in s.fifo.values()))
        fwd_box, bwd_box = new_fwd, new_bwd
        reports.append(rep)
    return reports, losses, grads


def run_lockstep(stages, batch_fn, n_mb: int, lr=0.0, record_grads=False):
    """Zero-delay reference: one micro-batch fully forward, then fully backward
    (each stage updating right after its backward), then the next micro-batch."""
    J = len(stages)
    for j, s in enumerate(stages, 1):
        s.j, s.J = j, J
    losses, grads = {}, {}
    for m in range(n_mb):
        lr_t = lr(m) if callable(lr) else lr
        for s in stages:
            s.lr = lr_t
        xs0, lab = batch_fn(m)
        msg = Fwd(m, list(xs0), lab)
        for s in stages[:-1]:
            msg = s.forward(msg)
        loss, b = stages[-1].tail_step(msg)
        losses[m] = loss
        if record_grads:
            grads[(J, m)] = stages[-1].last_grads
        for j in range(J - 1, 0, -1):
            b = stages[j - 1].backward(b)
            if record_grads:
                grads[(j, m)] = stages[j - 1].last_grads
    return losses, grads


def backprop_grads(units, xs0, labels):
    """Standard backpropagation (Eqs. 1-3): forward storing the
    graph, loss, then delta_j / Delta_j stage by stage from the last unit.
    Returns (loss, [grads per parameter in units order]).  No state is mutated
    except BN running stats (updated in this single forward, reading c10)."""
    xs = list(xs0)
    graphs = []
    for u in units[:-1]:
        xs, g = u.forward_graph(xs, update_stats=True)
        graphs.append(g)
    loss, tg = units[-1].loss_graph(xs, labels)
    ds, grads = units[-1].vjp(tg)
    for i in range(len(units) - 2, -1, -1):
        u = units[i]
        if u.reversible:
            ds, g = u.vjp(graphs[i], ds)
        else:
            ds, g = u.vjp(graphs[i], ds, need_dx=(i > 0))
        grads = g + grads
    return loss, grads


def backprop_train(units, batch_fn, n_mb: int, lr, opt: OptConfig):
    """Monolithic backprop trainer with the same optimizer: the J=1 / zero-delay
    reference trajectory."""
    params = [p for u in units for p in u.params()]
    v = [np.zeros_like(p) for (_, p, _) in params]
    acc = [np.zeros_like(p) for (_, p, _) in params]
    losses = {}
    t = 1
    for m in range(n_mb):
        lr_t = lr(m) if callable(lr) else lr
        xs0, lab = batch_fn(m)
        loss, grads = backprop_grads(units, xs0, lab)
        losses[m] = loss
        for a, g in zip(acc, grads):
            a += g / opt.k
        if t % opt.k == 0:
            for (_, p, decay), vv, a in zip(params, v, acc):
                sgd_step(p, vv, a, lr_t, opt, decay)
                a[...] = 0.0
        t += 1
    return losses, v
