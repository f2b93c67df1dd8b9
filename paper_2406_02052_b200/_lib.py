"""ctypes mirror of include/petra.h and the loader of the in-tree libpetra.so.

Argument marshalling only: every step of the PETRA tick runs in the CUDA
kernels of libpetra.so.  If the library is missing the import of the package
still works (so CPU-only tooling can inspect it) but every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libpetra.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "petra.h")

MAX_STAGES = 64
MAX_COMM = 16

FP32, BF16_TC = 0, 1
UNIT_REV, UNIT_DS, UNIT_STEM, UNIT_TAIL = 0, 1, 2, 3
CMP_INPUTS, CMP_STASH = 1, 2  # petra_stage_desc.compare_buffers (Table 3 comparison modes)
T_CONV_W, T_BN_GAMMA, T_BN_BETA, T_FC_W, T_FC_B, T_BN_RMEAN, T_BN_RVAR = range(7)
STATUS = {0: "PETRA_OK", 1: "PETRA_E_ARG", 2: "PETRA_E_SHAPE", 3: "PETRA_E_ODD_CHANNELS",
          4: "PETRA_E_EMPTY_BUFFER", 5: "PETRA_E_ORDER", 6: "PETRA_E_NONFINITE", 7: "PETRA_E_CUDA",
          8: "PETRA_E_NCCL", 9: "PETRA_E_OOM", 10: "PETRA_E_UNSUPPORTED"}


class PetraConv(C.Structure):
    _fields_ = [("cin", C.c_int32), ("cout", C.c_int32), ("ksize", C.c_int32), ("stride", C.c_int32)]


class PetraUnit(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dst_half", C.c_int32), ("n_layers", C.c_int32),
                ("layer", PetraConv * 3), ("proj", PetraConv * 2), ("maxpool", C.c_int32),
                ("classes", C.c_int32)]


class PetraStageDesc(C.Structure):
    _fields_ = [("n_units", C.c_int32), ("units", C.POINTER(PetraUnit)),
                ("batch", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32), ("in_c", C.c_int32),
                ("precision", C.c_int32), ("momentum", C.c_float), ("weight_decay", C.c_float),
                ("bn_momentum", C.c_float), ("bn_eps", C.c_float), ("nesterov", C.c_int32),
                ("accumulation_k", C.c_int32), ("fifo_capacity", C.c_int32), ("compare_buffers", C.c_int32)]


class PetraTensorInfo(C.Structure):
    _fields_ = [("unit", C.c_int32), ("part", C.c_int32), ("kind", C.c_int32), ("decay", C.c_int32),
                ("ndim", C.c_int32), ("shape", C.c_int32 * 4), ("offset", C.c_int64), ("count", C.c_int64)]


class PetraMemoryReport(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("total", "params", "optimizer", "shadows", "fifo", "fifo_live",
                                          "workspace", "cmp_inputs", "cmp_stash")]


class PetraTickReport(C.Structure):
    _fields_ = [("tick", C.c_int64), ("n_stages", C.c_int32),
                ("fwd_mb", C.c_int64 * MAX_STAGES), ("bwd_mb", C.c_int64 * MAX_STAGES),
                ("param_version", C.c_int64 * MAX_STAGES), ("fifo_depth", C.c_int64 * MAX_STAGES)]


TRANSPORT_NONE, TRANSPORT_NCCL, TRANSPORT_LOCAL = 0, 1, 2


class PetraPipelineDesc(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stages", C.POINTER(PetraStageDesc)),
                ("stage_rank", C.POINTER(C.c_int32)), ("rank", C.c_int32), ("world", C.c_int32),
                ("seed", C.c_uint64), ("transport", C.c_int32), ("nccl_id", C.c_void_p),
                ("local_group", C.c_int64), ("join_comm", C.c_int32), ("wire", C.c_int32)]


class PetraCommEntry(C.Structure):
    _fields_ = [("peer", C.c_int32), ("send", C.c_int32), ("ptr", C.c_void_p), ("bytes", C.c_int64)]


class PetraCommPlan(C.Structure):
    _fields_ = [("n", C.c_int32), ("e", PetraCommEntry * MAX_COMM)]


class PetraSchedMsg(C.Structure):
    _fields_ = [("peer", C.c_int32), ("send", C.c_int32), ("kind", C.c_int32), ("stage", C.c_int32),
                ("mb", C.c_int64)]


class PetraSchedMsgs(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", PetraSchedMsg * 8)]


class PetraConvGeom(C.Structure):
    _fields_ = [("batch", C.c_int32), ("h", C.c_int32), ("w", C.c_int32), ("cin", C.c_int32),
                ("cout", C.c_int32), ("ksize", C.c_int32), ("stride", C.c_int32)]


class PetraProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


P, VP, I32, I64, U64, F32 = C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float
SIGS = {
    "petra_status_str": (C.c_char_p, [C.c_int]),
    "petra_last_error": (C.c_char_p, []),
    "petra_version": (C.c_char_p, []),
    "petra_stage_create": (C.c_int, [C.POINTER(PetraStageDesc), U64, C.POINTER(P)]),
    "petra_stage_destroy": (C.c_int, [P]),
    "petra_stage_output_shape": (C.c_int, [P, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)]),
    "petra_stage_param_count": (C.c_int, [P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "petra_stage_memory": (C.c_int, [P, C.POINTER(PetraMemoryReport)]),
    "petra_stage_eval": (C.c_int, [P, VP, VP, VP, VP, VP]),
    "petra_stage_eval_tail": (C.c_int, [P, VP, VP, VP, VP, VP, VP]),
    "petra_stage_num_tensors": (C.c_int, [P, C.POINTER(I32)]),
    "petra_stage_tensor_info": (C.c_int, [P, I32, C.POINTER(PetraTensorInfo)]),
    "petra_stage_get_params": (C.c_int, [P, VP, VP, VP]),
    "petra_stage_set_params": (C.c_int, [P, VP, VP, VP]),
    "petra_stage_get_grads": (C.c_int, [P, VP]),
    "petra_stage_forward": (C.c_int, [P, U64, VP, VP, VP, VP, VP]),
    "petra_stage_backward": (C.c_int, [P, U64, VP, VP, VP, VP, VP, VP, VP, VP, F32, VP]),
    "petra_stage_tail": (C.c_int, [P, U64, VP, VP, VP, F32, VP, VP, VP, VP, VP, VP]),
    "petra_pipeline_create": (C.c_int, [C.POINTER(PetraPipelineDesc), C.POINTER(P)]),
    "petra_pipeline_destroy": (C.c_int, [P]),
    "petra_nccl_unique_id": (C.c_int, [VP]),
    "petra_set_allocator": (C.c_int, [VP, VP, VP]),
    "petra_pipeline_stage": (C.c_int, [P, I32, C.POINTER(P)]),
    "petra_pipeline_tick": (C.c_int, [P, I64, I32, VP, VP, F32, VP, VP, C.POINTER(PetraTickReport)]),
    "petra_pipeline_comm": (C.c_int, [P, I64, C.POINTER(PetraCommPlan)]),
    "petra_pipeline_timing": (C.c_int, [P, I32]),
    "petra_pipeline_stage_ms": (C.c_int, [P, C.POINTER(C.c_float), I32, C.POINTER(I32)]),
    "petra_schedule_create": (C.c_int, [I32, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32), I32, C.POINTER(P)]),
    "petra_schedule_tick": (C.c_int, [P, I64, I32, C.POINTER(PetraTickReport), C.POINTER(PetraSchedMsgs)]),
    "petra_schedule_destroy": (C.c_int, [P]),
    "petra_conv_run": (C.c_int, [I32, I32, C.POINTER(PetraConvGeom), VP, VP, VP, VP]),
    "petra_conv_engine": (C.c_int32, [C.POINTER(PetraConvGeom), I32, I32]),
    "petra_conv_bn_stats": (C.c_int, [C.POINTER(PetraConvGeom), I32, VP, VP, VP, VP, VP]),
    "petra_conv_plan": (C.c_int, [C.POINTER(PetraConvGeom), I32, C.POINTER(I32)]),
    "petra_conv_bench": (I32, [I32, I32, C.POINTER(PetraConvGeom), I32, I32, C.POINTER(C.c_float)]),
    "petra_launch_count": (C.c_int64, []),
    "petra_profile": (C.c_int, [I32]),
    "petra_profile_read": (C.c_int, [C.POINTER(PetraProfEntry), I32, C.POINTER(I32)]),
    "petra_profile_records": (C.c_int, [VP, I32, C.POINTER(I32)]),
}


def launch_count() -> int:
    return int(lib().petra_launch_count())


def profile(enable: bool):
    call("petra_profile", int(bool(enable)))


class PetraProfRecord(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("ms", C.c_float), ("flops", C.c_double), ("bytes", C.c_double),
                ("ctas", C.c_int32)]


def profile_records():
    """Per logical kernel of the profiled replay: name, event ms, algorithmic flops and bytes."""
    n = C.c_int32()
    one = (PetraProfRecord * 1)()
    call("petra_profile_records", C.cast(one, C.c_void_p), 0, C.byref(n))
    arr = (PetraProfRecord * max(1, n.value))()
    call("petra_profile_records", C.cast(arr, C.c_void_p), n.value, C.byref(n))
    return [dict(name=arr[i].name.decode(), ms=arr[i].ms, flops=arr[i].flops, bytes=arr[i].bytes,
                 ctas=arr[i].ctas) for i in range(n.value)]


def profile_read():
    arr = (PetraProfEntry * 64)()
    n = C.c_int32()
    call("petra_profile_read", arr, 64, C.byref(n))
    return [dict(name=arr[i].name.decode(), launches=arr[i].launches, ms=arr[i].ms, flops=arr[i].flops,
                 bytes=arr[i].bytes) for i in range(n.value)]


class PetraError(RuntimeError):
    def __init__(self, status, fn, detail):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{fn}: {self.name}: {detail}")


_lib = None


def header_functions():
    """Names of the functions declared in include/petra.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(petra_[a-z_]+)\s*\(", txt)))


def lib():
    """The loaded libpetra.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2406_02052_b200.build` "
                              "(there is no CPU fallback)")
        l = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def call(name, *args):
    """Call an ABI function and raise PetraError on a non-OK status."""
    st = getattr(lib(), name)(*args)
    if st != 0:
        raise PetraError(st, name, lib().petra_last_error().decode())
    return st
