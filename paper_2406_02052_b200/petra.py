"""Thin Python binding over libpetra.so: same names as the C ABI, torch CUDA
tensors in, pointers out.  No arithmetic happens here."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .models import StageSpec


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor expected (libpetra has no CPU path)")
    if not t.is_contiguous():
        raise ValueError("contiguous tensor expected")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Stage:
    """petra_stage_* : one PETRA stage on the current CUDA device."""

    def __init__(self, spec: StageSpec = None, seed: int = 0, _handle=None):
        self._owned = _handle is None
        if _handle is None:
            self._desc, self._arr = spec.to_c()
            h = C.c_void_p()
            L.call("petra_stage_create", C.byref(self._desc), seed, C.byref(h))
            self.h = h
        else:
            self.h = _handle
        np_, nb = C.c_size_t(), C.c_size_t()
        L.call("petra_stage_param_count", self.h, C.byref(np_), C.byref(nb))
        self.n_params, self.n_buffers = np_.value, nb.value
        n = C.c_int32()
        L.call("petra_stage_num_tensors", self.h, C.byref(n))
        self.tensors = []
        for i in range(n.value):
            ti = L.PetraTensorInfo()
            L.call("petra_stage_tensor_info", self.h, i, C.byref(ti))
            self.tensors.append(dict(unit=ti.unit, part=ti.part, kind=ti.kind, decay=ti.decay,
                                     shape=tuple(ti.shape[:ti.ndim]), offset=ti.offset, count=ti.count))
        b, hh, w, c = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        L.call("petra_stage_output_shape", self.h, C.byref(b), C.byref(hh), C.byref(w), C.byref(c))
        self.out_shape = (b.value, hh.value, w.value, c.value)

    def close(self):
        if self._owned and self.h:
            L.call("petra_stage_destroy", self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- parameters (host numpy float32)
    def get_params(self):
        th = np.zeros(self.n_params, np.float32)
        v = np.zeros(self.n_params, np.float32)
        bf = np.zeros(max(1, self.n_buffers), np.float32)
        L.call("petra_stage_get_params", self.h, th.ctypes.data, v.ctypes.data, bf.ctypes.data)
        return th, v, bf[:self.n_buffers]

    def set_params(self, theta=None, v=None, buffers=None):
        cv = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
        th, vv, bf = cv(theta), cv(v), cv(buffers)
        L.call("petra_stage_set_params", self.h, None if th is None else th.ctypes.data,
               None if vv is None else vv.ctypes.data, None if bf is None else bf.ctypes.data)

    def memory(self):
        """petra_stage_memory: device bytes by category (Table 3 accounting)."""
        r = L.PetraMemoryReport()
        L.call("petra_stage_memory", self.h, C.byref(r))
        return {n: getattr(r, n) for n, _ in L.PetraMemoryReport._fields_}

    def get_grads(self):
        g = np.zeros(self.n_params, np.float32)
        L.call("petra_stage_get_grads", self.h, g.ctypes.data)
        return g

    # ---- ticks (torch CUDA fp32 tensors, NHWC halves)
    def forward(self, mb, x1, x2, o1, o2, stream=None):
        L.call("petra_stage_forward", self.h, mb, _ptr(x1), _ptr(x2), _ptr(o1), _ptr(o2), _stream(stream))

    def backward(self, mb, xt1, xt2, d1, d2, oxt1, oxt2, od1, od2, lr, stream=None):
        L.call("petra_stage_backward", self.h, mb, _ptr(xt1), _ptr(xt2), _ptr(d1), _ptr(d2), _ptr(oxt1),
               _ptr(oxt2), _ptr(od1), _ptr(od2), float(lr), _stream(stream))

    def tail(self, mb, x1, x2, labels, lr, oxt1, oxt2, od1, od2, loss, stream=None):
        L.call("petra_stage_tail", self.h, mb, _ptr(x1), _ptr(x2), _ptr(labels), float(lr), _ptr(oxt1),
               _ptr(oxt2), _ptr(od1), _ptr(od2), _ptr(loss), _stream(stream))

    def eval(self, x1, x2, o1, o2, stream=None):
        """petra_stage_eval: forward with BN on the running statistics (no state change)."""
        L.call("petra_stage_eval", self.h, _ptr(x1), _ptr(x2), _ptr(o1), _ptr(o2), _stream(stream))

    def eval_tail(self, x1, x2, labels, correct, loss, stream=None):
        """petra_stage_eval_tail: evaluation forward + classifier; correct (int32[1]) += hits."""
        L.call("petra_stage_eval_tail", self.h, _ptr(x1), _ptr(x2), _ptr(labels), _ptr(correct), _ptr(loss),
               _stream(stream))


def report_dict(rep: L.PetraTickReport):
    J = rep.n_stages
    return dict(tick=rep.tick, fwd_mb=list(rep.fwd_mb[:J]), bwd_mb=list(rep.bwd_mb[:J]),
                version=list(rep.param_version[:J]), fifo_depth=list(rep.fifo_depth[:J]))


class Pipeline:
    """petra_pipeline_* : the stages of this rank with double-buffered mailboxes."""

    def __init__(self, specs, stage_rank=None, rank=0, world=1, seed=0, transport="none", nccl_id=None,
                 local_group=0, join_comm=True, wire="fp32"):
        """transport: "none" (world 1, or the caller moves petra_pipeline_comm's bytes),
        "nccl" (the library's ncclSend/ncclRecv; nccl_id = nccl_unique_id() of rank 0),
        "local" (ranks = pipelines of this process sharing local_group; a test transport).
        wire: "fp32" or "bf16" (petra_wire: messages rounded to bf16 at every stage boundary)."""
        J = len(specs)
        self.J = J
        self._keep = [s.to_c() for s in specs]
        descs = (L.PetraStageDesc * J)(*[d for d, _ in self._keep])
        sr = (C.c_int32 * J)(*(stage_rank or [0] * J))
        tr = {"none": L.TRANSPORT_NONE, "nccl": L.TRANSPORT_NCCL, "local": L.TRANSPORT_LOCAL}[transport]
        self._nid = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        pd = L.PetraPipelineDesc(J, C.cast(descs, C.POINTER(L.PetraStageDesc)), C.cast(sr, C.POINTER(C.c_int32)),
                                 rank, world, seed, tr, C.cast(self._nid, C.c_void_p) if self._nid else None,
                                 int(local_group), int(bool(join_comm)), {"fp32": 0, "bf16": 1}[wire])
        self._descs, self._sr = descs, sr
        h = C.c_void_p()
        L.call("petra_pipeline_create", C.byref(pd), C.byref(h))
        self.h = h
        self.stages = {}
        for j in range(1, J + 1):
            sh = C.c_void_p()
            L.call("petra_pipeline_stage", self.h, j, C.byref(sh))
            if sh.value:
                self.stages[j] = Stage(_handle=sh)

    def close(self):
        if self.h:
            for s in self.stages.values():
                s.h = None
            L.call("petra_pipeline_destroy", self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tick(self, t, inject, x0=None, labels=None, lr=0.0, loss=None, stream=None, report=True):
        rep = L.PetraTickReport() if report else None
        L.call("petra_pipeline_tick", self.h, t, int(bool(inject)), _ptr(x0), _ptr(labels), float(lr), _ptr(loss),
               _stream(stream), C.byref(rep) if report else None)
        return report_dict(rep) if report else None

    def timing(self, on=True):
        L.call("petra_pipeline_timing", self.h, int(bool(on)))

    def stage_ms(self):
        arr = (C.c_float * self.J)()
        n = C.c_int32()
        L.call("petra_pipeline_stage_ms", self.h, arr, self.J, C.byref(n))
        return [arr[i] / max(n.value, 1) for i in range(self.J)]

    def comm(self, t):
        plan = L.PetraCommPlan()
        L.call("petra_pipeline_comm", self.h, t, C.byref(plan))
        return [(plan.e[i].peer, plan.e[i].send, plan.e[i].ptr, plan.e[i].bytes) for i in range(plan.n)]


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)
_RELEASE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_void_p)
_allocator_keep = []


def use_torch_allocator(enable: bool = True):
    """petra_set_allocator with PyTorch's caching allocator (enable) or cudaMalloc (not):
    the library's parameters, FIFOs and workspace then live in torch's pool."""
    import torch
    if not enable:
        L.call("petra_set_allocator", None, None, None)
        return

    def alloc(n, dev, ctx):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(n), int(dev)))
        except Exception:
            return None

    def release(p, dev, ctx):
        torch.cuda.caching_allocator_delete(int(p))
    fa, fr = _ALLOC_FN(alloc), _RELEASE_FN(release)
    _allocator_keep[:] = [fa, fr]  # the library holds raw pointers to the callbacks
    L.call("petra_set_allocator", C.cast(fa, C.c_void_p), C.cast(fr, C.c_void_p), None)


def nccl_unique_id() -> bytes:
    """petra_nccl_unique_id: 128 bytes for PETRA_TRANSPORT_NCCL (create on rank 0, share)."""
    buf = C.create_string_buffer(128)
    L.call("petra_nccl_unique_id", buf)
    return buf.raw


class Schedule:
    """petra_schedule_* : the host-only integer bookkeeping of the pipeline."""

    def __init__(self, stage_rank, nonrev, rank=0, accum_k=None):
        J = len(stage_rank)
        sr = (C.c_int32 * J)(*stage_rank)
        nr = (C.c_int32 * J)(*nonrev)
        ks = (C.c_int32 * J)(*accum_k) if accum_k is not None else None
        h = C.c_void_p()
        L.call("petra_schedule_create", J, sr, nr, ks, rank, C.byref(h))
        self.h = h

    def tick(self, t, inject):
        rep, msgs = L.PetraTickReport(), L.PetraSchedMsgs()
        L.call("petra_schedule_tick", self.h, t, int(bool(inject)), C.byref(rep), C.byref(msgs))
        ms = [dict(peer=msgs.m[i].peer, send=msgs.m[i].send, kind=msgs.m[i].kind, stage=msgs.m[i].stage,
                   mb=msgs.m[i].mb) for i in range(msgs.n)]
        return report_dict(rep), ms

    def __del__(self):
        try:
            if self.h:
                L.call("petra_schedule_destroy", self.h)
        except Exception:
            pass
