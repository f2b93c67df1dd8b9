"""torchrun worker for tests/test_multirank_nccl_gpu.py (one rank per GPU).

Every rank runs the world-N pipeline with the library's NCCL transport
(PETRA_TRANSPORT_NCCL: ncclSend / ncclRecv on library-owned streams) and, on its own
GPU, the world-1 pipeline of the same model and inputs; the stages it owns must be
bitwise equal to world 1's (the rank layout adds no arithmetic, reading c14)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import models as OM  # noqa: E402
from paper_2406_02052_b200 import Pipeline, petra, _lib as L, models as PM  # noqa: E402
from paper_2406_02052_b200.dist import contiguous_stage_ranks  # noqa: E402
from tests.gpu_harness import nhwc, oracle_to_product_units, pack_params, rand_params  # noqa: E402


def run(pipe, sr, rank, B, n_mb, J, lr=0.025):
    loss = torch.zeros(1, device="cuda")
    losses = {}
    for t in range(n_mb + 2 * J - 2):
        inject = t < n_mb
        x0 = lab = None
        if inject and sr[0] == rank:
            x = synth.images((B, 3, 32, 32), 0, t)
            x0 = torch.tensor(nhwc(x), dtype=torch.float32, device="cuda")
            lab = torch.tensor(synth.labels(B, 10, 0, t), dtype=torch.int32, device="cuda")
        rep = pipe.tick(t, inject, x0, lab, lr, loss if sr[-1] == rank else None)
        if sr[-1] == rank:
            torch.cuda.synchronize()
            if rep["fwd_mb"][-1] >= 0:
                losses[rep["fwd_mb"][-1]] = loss.item()
    torch.cuda.synchronize()
    return losses


def main():
    os.environ.setdefault("PETRA_STAGES_PER_GPU", "4")  # same kernel plans on every rank layout
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    B, n_mb, counts = 8, 6, [5, 4, 4, 5]
    J = len(counts)
    units = rand_params(OM.build_revnet("revnet18", 32, 10), 5)
    init = [pack_params(g) for g in OM.group(units, counts)]
    specs = PM.stage_specs(oracle_to_product_units(units), counts, B, (32, 32, 3), L.BF16_TC)
    nid = [petra.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(nid, src=0)
    sr = contiguous_stage_ranks(J, world)
    pipe = Pipeline(specs, sr, rank, world, seed=0, transport="nccl", nccl_id=nid[0])
    ref = Pipeline(specs, [0] * J, 0, 1, seed=0)
    for p in (pipe, ref):
        for j, s in p.stages.items():
            th, bf = init[j - 1]
            s.set_params(th, np.zeros_like(th), bf)
    lw = run(pipe, sr, rank, B, n_mb, J)
    l1 = run(ref, [0] * J, 0, B, n_mb, J)
    ok = True
    if sr[-1] == rank:
        ok &= lw == l1
    for j, s in pipe.stages.items():
        for a, b in zip(s.get_params(), ref.stages[j].get_params()):
            ok &= bool(np.array_equal(a, b))
    print(f"rank {rank}: stages {sorted(pipe.stages)} bitwise equal to world 1: {ok}", flush=True)
    pipe.close()
    ref.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
