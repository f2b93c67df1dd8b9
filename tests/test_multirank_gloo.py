"""World-size-2 test of the multi-rank PETRA routing on CPU (gloo).

Each rank owns a contiguous block of stages (contiguous_stage_ranks, the map
bench.py uses), follows the C-ABI host schedule (petra_schedule_tick -- the
same bookkeeping petra_pipeline_tick runs on the GPU) to decide what its
stages do at each tick and which messages cross the rank boundary, computes
the stages with the fp64 oracle, and moves the messages with torch.distributed
point-to-point ops over gloo.  The result must equal the single-process PETRA
run bitwise: the transport and schedule add no arithmetic.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

J, T, B = 4, 5, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _build():
    from tests.test_oracle_engine import chain, make_stages
    groups, _ = chain(J, "dr")
    return groups, make_stages(groups)


def _batch(m):
    from tests.test_oracle_engine import batch_fn
    return batch_fn(m)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import engine as E
    from oracle import models as OM
    from paper_2406_02052_b200 import Schedule
    from paper_2406_02052_b200.dist import contiguous_stage_ranks

    groups, stages = _build()
    for j, s in enumerate(stages, 1):
        s.j, s.J = j, J
    stage_rank = contiguous_stage_ranks(J, world)
    nonrev = [sum(1 for u in g if not u.reversible and not getattr(u, "is_tail", False)) for g in groups]
    sched = Schedule(stage_rank, nonrev, rank)
    local = [j for j in range(1, J + 1) if stage_rank[j - 1] == rank]
    # message shapes (NCHW halves) at every stage boundary
    shapes = [[(B, 3, 4, 4)]]
    for g in groups[:-1]:
        _, sh = OM.stage_shapes(g, shapes[-1])
        shapes.append(sh)
    fwd = {j: [None, None] for j in local}
    bwd = {j: [None, None] for j in local}
    ghost_f, ghost_b = [None, None], [None, None]
    for t in range(T + 2 * J - 2):
        rep, msgs = sched.tick(t, t < T)
        p, q = t & 1, (t - 1) & 1
        for j in local:
            fmb, bmb = rep["fwd_mb"][j - 1], rep["bwd_mb"][j - 1]
            s = stages[j - 1]
            s.lr = 0.05
            fin = None
            if fmb >= 0:
                if j == 1:
                    xs, y = _batch(fmb)
                    fin = E.Fwd(fmb, xs, y)
                else:
                    fin = fwd[j - 1][q] if (j - 1) in fwd else ghost_f[q]
                    assert fin.mb == fmb
            if j < J:
                fwd[j][p] = s.forward(fin) if fin is not None else None
                if bmb >= 0:
                    bin_ = bwd[j + 1][q] if (j + 1) in bwd else ghost_b[q]
                    assert bin_.mb == bmb
                    bwd[j][p] = s.backward(bin_)
                else:
                    bwd[j][p] = None
            else:
                bwd[j][p] = s.tail_step(fin)[1] if fin is not None else None
        # transport: one batched group of isend / irecv
        ops, recv_f, recv_b = [], None, None
        for m in msgs:
            j = m["stage"]
            if m["kind"] == 0:
                if m["send"]:
                    msg = fwd[j][p]
                    ts = [torch.from_numpy(np.ascontiguousarray(x)) for x in msg.xs] + [torch.from_numpy(msg.labels)]
                else:
                    ts = [torch.empty(sh, dtype=torch.float64) for sh in shapes[j]] + [torch.empty(B, dtype=torch.int64)]
                    recv_f = (m["mb"], ts)
            else:
                if m["send"]:
                    msg = bwd[j][p]
                    ts = [torch.from_numpy(np.ascontiguousarray(x)) for x in msg.xs + msg.ds]
                else:
                    sh = shapes[j - 1]
                    ts = [torch.empty(s_, dtype=torch.float64) for s_ in sh + sh]
                    recv_b = (m["mb"], ts)
            for x in ts:
                ops.append(dist.P2POp(dist.isend if m["send"] else dist.irecv, x, m["peer"]))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        ghost_f[p] = None if recv_f is None else E.Fwd(recv_f[0], [x.numpy() for x in recv_f[1][:2]],
                                                       recv_f[1][2].numpy())
        ghost_b[p] = None if recv_b is None else E.Bwd(recv_b[0], [x.numpy() for x in recv_b[1][:2]],
                                                       [x.numpy() for x in recv_b[1][2:]])
    out[rank] = {j: [p_.copy() for (_, p_, _) in stages[j - 1].params()] for j in local}
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_pipeline_equals_single_process():
    from oracle import engine as E
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, start_method="spawn", join=True)
    groups, stages = _build()
    E.run_petra(stages, _batch, T, lr=0.05)
    got = {}
    for r in range(2):
        got.update(out[r])
    assert sorted(got) == list(range(1, J + 1))
    for j in range(1, J + 1):
        want = [p for (_, p, _) in stages[j - 1].params()]
        for a, b in zip(got[j], want):
            assert np.array_equal(a, b), j
