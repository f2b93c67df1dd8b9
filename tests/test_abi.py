"""CPU-side checks of the C-ABI library (no compute calls without a GPU):
exports, error paths, the host-only schedule against the oracle's tick engine
(bit-exact integers), and the product model builder against the oracle's."""
import ctypes as C
import subprocess

import numpy as np
import pytest
import torch

from oracle import engine as E
from oracle import models as OM
from oracle.units import DSUnit, RevUnit, StemUnit, TailUnit
from paper_2406_02052_b200 import Schedule, _lib as L, models as PM


def test_library_exports_every_header_symbol():
    declared = L.header_functions()
    assert len(declared) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    lib = L.lib()
    for f in declared:
        assert hasattr(lib, f)
    assert b"sm_100a" in lib.petra_version()


def test_status_strings_and_no_fallback():
    lib = L.lib()
    assert lib.petra_status_str(0) == b"ok"
    assert lib.petra_status_str(7) == b"CUDA error"
    if torch.cuda.is_available():
        pytest.skip("no-device error path only checkable without a GPU")
    spec = PM.stage_specs(PM.revnet("revnet18"), [5, 4, 4, 5], 2, (32, 32, 3))[1]
    d, arr = spec.to_c()
    h = C.c_void_p()
    st = lib.petra_stage_create(C.byref(d), 0, C.byref(h))
    assert st == 7 and b"no CPU fallback" in lib.petra_last_error()


def test_null_arguments_are_rejected():
    lib = L.lib()
    assert lib.petra_stage_create(None, 0, None) == 1
    assert lib.petra_stage_forward(None, 0, None, None, None, None, None) == 1
    assert lib.petra_pipeline_tick(None, 0, 0, None, None, 0.0, None, None, None) == 1
    assert lib.petra_schedule_create(0, None, None, None, 0, None) == 1


@pytest.mark.parametrize("J", [1, 2, 4, 10])
def test_schedule_matches_oracle_engine(J):
    """petra_schedule (the bookkeeping petra_pipeline_tick runs) vs the oracle's
    tick engine run on real (tiny) oracle stages: bit-exact integer reports."""
    from tests.test_oracle_engine import batch_fn, chain, make_stages
    if J == 1:
        groups = [[u for g in chain(3, "r")[0] for u in g]]
    else:
        groups, _ = chain(J, "rdr")
    stages = make_stages(groups)
    T = 6
    reps, _, _ = E.run_petra(stages, batch_fn, T, lr=0.01)
    nonrev = [sum(1 for u in g if not u.reversible and not getattr(u, "is_tail", False)) for g in groups]
    s = Schedule([0] * J, nonrev)
    for r in reps:
        got, msgs = s.tick(r.tick, r.tick < T)
        assert got["fwd_mb"] == r.fwd_mb and got["bwd_mb"] == r.bwd_mb, (r, got)
        assert got["version"] == r.version and got["fifo_depth"] == r.fifo_depth, (r, got)
        assert msgs == []  # single rank: no transport


@pytest.mark.parametrize("ks", [[2, 2, 2, 2], [1, 3, 2, 4]])
def test_schedule_accumulation_matches_oracle_engine(ks):
    """Accumulation k > 1 (Alg. 1 lines 19-23): the schedule's param_version is
    the oracle stages' update count, bit-exact, with a different k per stage."""
    from tests.test_oracle_engine import batch_fn, chain
    groups, _ = chain(4, "rdr")
    stages = [E.Stage(g, E.OptConfig(k=k)) for g, k in zip(groups, ks)]
    T = 9
    reps, _, _ = E.run_petra(stages, batch_fn, T, lr=0.01)
    nonrev = [sum(1 for u in g if not u.reversible and not getattr(u, "is_tail", False)) for g in groups]
    s = Schedule([0] * 4, nonrev, accum_k=ks)
    for r in reps:
        got, _ = s.tick(r.tick, r.tick < T)
        assert got["version"] == r.version and got["fwd_mb"] == r.fwd_mb, (r, got)
    assert [st.version for st in stages] == [(T // k) for k in ks]


def test_schedule_comm_plan_two_ranks():
    """Every message the sender lists after tick t is listed by the receiver
    with the same (stage, kind, mb), and it is consumed at t+1."""
    J, T = 4, 5
    ranks = [0, 0, 1, 1]
    scheds = [Schedule(ranks, [1, 1, 0, 0], r) for r in range(2)]
    for t in range(T + 2 * J - 2):
        plans = [s.tick(t, t < T)[1] for s in scheds]
        sends = sorted((m["stage"], m["kind"], m["mb"]) for r, p in enumerate(plans) for m in p if m["send"])
        recvs = sorted((m["stage"], m["kind"], m["mb"]) for r, p in enumerate(plans) for m in p if not m["send"])
        assert sends == recvs
        for r, p in enumerate(plans):
            for m in p:
                assert m["peer"] == 1 - r


def test_product_models_match_oracle_architecture():
    """The product's RevNet builder describes the same layers as the oracle's
    (independently written) builder, and the partitioner covers all units."""
    for name, H, classes in (("revnet18", 32, 10), ("revnet34", 32, 1000), ("revnet50", 224, 1000)):
        pu = PM.revnet(name, H, classes)
        ou = OM.build_revnet(name, H, classes)
        assert len(pu) == len(ou)
        for p, o in zip(pu, ou):
            if isinstance(o, RevUnit):
                assert p.kind == L.UNIT_REV and p.dst == o.dst
                assert p.layers == [(l.cin, l.cout, l.k, l.stride) for l in o.phi.layers]
            elif isinstance(o, DSUnit):
                assert p.kind == L.UNIT_DS
                assert p.layers == [(l.cin, l.cout, l.k, l.stride) for l in o.phi.layers]
                assert p.proj == [(q.cin, q.cout, q.k, q.stride) for q in (o.pa, o.pb)]
            elif isinstance(o, StemUnit):
                assert p.kind == L.UNIT_STEM and p.maxpool == int(o.maxpool)
            elif isinstance(o, TailUnit):
                assert p.kind == L.UNIT_TAIL and p.classes == o.classes
        for J in (1, 2, 4, 8, 16):
            counts = PM.partition(pu, J, 64, H, H, 3)
            assert len(counts) == J and sum(counts) == len(pu) and min(counts) >= 1


def test_partition_is_flop_balanced():
    pu = PM.revnet("revnet18", 32, 10)
    counts = PM.partition(pu, 4)
    cost = PM.conv_macs(pu, 64, 32, 32, 3)
    i, per = 0, []
    for c in counts:
        per.append(sum(cost[i:i + c]))
        i += c
    assert max(per) <= 1.25 * sum(cost) / 4


def test_set_allocator_argument_checks():
    """petra_set_allocator: alloc and release go together; (NULL, NULL) restores cudaMalloc.
    Host-only (no device work)."""
    import ctypes as C
    from paper_2406_02052_b200 import _lib as L
    fa = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)(lambda n, d, c: None)
    assert L.lib().petra_set_allocator(C.cast(fa, C.c_void_p), None, None) == 1  # PETRA_E_ARG
    assert L.lib().petra_set_allocator(None, None, None) == 0
