"""PETRA (arXiv 2406.02052) fp64 CPU oracle.

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call or execute anything under
``oracle/``.  The CUDA path (``paper_2406_02052_b200``) never imports it, and
the two share no code: no kernels, headers, helpers, tables or constant
generators.  Only the seeded input generators in ``synth/`` serve both.

Parity status:
  * primitives (conv, BN, ReLU, max-pool, linear, CE) -- pinned by worked
    examples, brute force, torch.nn.functional fp64, finite differences;
  * units (coupling forward / inverse / VJP) -- pinned by the worked scalar
    example, frozen-theta exact inversion, FD, torch.autograd fp64;
  * engine (tick schedule, FIFO, updates) -- pinned by the closed-form
    schedule of Table 1 (delay 2(J-j)), J=1 == backprop, lockstep == backprop,
    lr=0 gradient equality, torch.optim.SGD(nesterov=True);
  * trained accuracy (Table 2) -- parity unpinned (needs datasets; out of scope).
"""
from . import primitives, units, engine, models  # noqa: F401
