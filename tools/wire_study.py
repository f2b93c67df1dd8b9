"""bf16 wire format (petra_wire): error growth against the fp32 wire.

Runs the bench pipeline (RevNet-18, CIFAR shape, batch 64, J = 4; one GPU) three ways from
the same seeds and data for T ticks:
  A  bf16 tensor-core convolutions, fp32 wire  (the bench configuration)
  B  bf16 tensor-core convolutions, bf16 wire  (every message rounded to bf16)
  C  fp32 convolutions, fp32 wire              (the precision reference)
and prints, every few ticks, rel ||theta_B - theta_A|| / ||theta_A|| (what the wire adds)
next to rel ||theta_A - theta_C|| / ||theta_C|| (what the bf16 tensor-core path already
costs), and the losses.  Product code only (no oracle).
    python tools/wire_study.py [ticks] > profiles/r02/wire_bf16.json
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02052_b200 import Pipeline, _lib as L, models as PM  # noqa: E402


def run(precision, wire, T, B=64, J=4, every=5):
    torch.cuda.set_device(0)
    units = PM.revnet("revnet18", 32, 10)
    counts = PM.partition(units, J, B, 32, 32, 3)
    specs = PM.stage_specs(units, counts, B, (32, 32, 3), precision, 5e-4)
    pipe = Pipeline(specs, [0] * J, 0, 1, seed=1, wire=wire)
    gen = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn((B, 32, 32, 3), generator=gen, device="cuda") for _ in range(16)]
    ys = [torch.randint(0, 10, (B,), generator=gen, device="cuda", dtype=torch.int32) for _ in range(16)]
    loss = torch.zeros(1, device="cuda")
    thetas, losses = {}, {}
    for t in range(T):
        pipe.tick(t, True, xs[t % 16], ys[t % 16], 0.025, loss, report=False)
        torch.cuda.synchronize()
        if t >= 2 * J - 2:
            losses[t] = loss.item()
        if (t + 1) % every == 0:
            thetas[t] = np.concatenate([s.get_params()[0] for _, s in sorted(pipe.stages.items())])
    pipe.close()
    return thetas, losses


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    A = run(L.BF16_TC, "fp32", T)
    Bw = run(L.BF16_TC, "bf16", T)
    C = run(L.FP32, "fp32", T)
    rows = []
    for t in sorted(A[0]):
        ta, tb, tc = A[0][t], Bw[0][t], C[0][t]
        rows.append({"tick": t, "wire_rel_theta": float(np.linalg.norm(tb - ta) / np.linalg.norm(ta)),
                     "bf16_path_rel_theta": float(np.linalg.norm(ta - tc) / np.linalg.norm(tc)),
                     "loss_fp32_wire": A[1].get(t), "loss_bf16_wire": Bw[1].get(t), "loss_fp32_path": C[1].get(t)})
    print(json.dumps({"workload": "RevNet-18, CIFAR shape, batch 64, J=4, one GPU, lr 0.025, synthetic data",
                      "ticks": T, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
