"""Cross-rank transport of PETRA messages (product side plumbing).

After every tick the pipeline lists the device buffers this rank must send to
or receive from its neighbours (petra_pipeline_comm); they are moved with one
batched NCCL send/recv group through torch.distributed (NVLink / NVSwitch on a
B200 box).  Neighbour-only point-to-point traffic, no collective (SURVEY.md
8(e)): forward messages carry 2 activation halves + labels, backward messages
the reconstructed input halves + the 2 gradient halves ("backward
communication by a factor of 4").
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _Raw:
    """Zero-copy view of a raw device allocation as a uint8 torch tensor."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def raw_tensor(ptr, nbytes):
    return torch.as_tensor(_Raw(ptr, nbytes), device="cuda")


class Transport:
    def __init__(self, pipeline):
        self.p = pipeline
        self._cache = {}

    def _t(self, ptr, nbytes):
        key = (ptr, nbytes)
        if key not in self._cache:
            self._cache[key] = raw_tensor(ptr, nbytes)
        return self._cache[key]

    def exchange(self, t):
        """Move the messages produced at tick t (to be consumed at t+1)."""
        plan = self.p.comm(t)
        if not plan:
            return
        ops = []
        for peer, send, ptr, nbytes in plan:
            op = dist.isend if send else dist.irecv
            ops.append(dist.P2POp(op, self._t(ptr, nbytes), peer))
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def contiguous_stage_ranks(J: int, world: int):
    """Contiguous map of J stages onto `world` ranks (J/world each, first ranks
    take the remainder)."""
    if world > J:
        raise ValueError(f"{world} ranks for {J} stages")
    base, rem = divmod(J, world)
    out = []
    for r in range(world):
        out += [r] * (base + (1 if r < rem else 0))
    return out
