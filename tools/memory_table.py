"""Table 3 of the paper for this implementation, MEASURED: device memory
of RevNet-50 on ImageNet-shaped input, batch 64, one stage per residual block (J = 18,
PAPER.md:259), in the four configurations the paper compares -- each one a real pipeline
whose stages allocate (and every tick write) the buffers of that configuration:

  input buffer  (delayed-gradient methods, PipeDream): every stage j >= 2 keeps the inputs of
                its 2(J-j)+1 in-flight micro-batches (petra_stage_desc.compare_buffers bit
                PETRA_CMP_INPUTS; PETRA itself buffers only the inputs of its non-reversible
                units); the first stage's is excluded, as in the paper (its input is the data);
  param buffer  (weight stashing, PipeDream): 2(J-j) extra fp32 copies of theta_j, one written
                every forward (PETRA_CMP_STASH).

Per configuration: the pipeline runs 2J ticks (so every ring slot is written), then the
stages' petra_stage_memory reports are summed and the device footprint is read as the drop
in cudaMemGetInfo free bytes across the pipeline's lifetime (creation .. after the ticks).
Needs a GPU.  Prints one JSON object.
    python tools/memory_table.py [--model revnet50] [--stages 0] [--batch 64] [--ticks -1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2406_02052_b200 import Pipeline  # noqa: E402
from paper_2406_02052_b200 import _lib as L  # noqa: E402
from paper_2406_02052_b200 import models as PM  # noqa: E402

IMAGE = {"revnet18": 32, "revnet34": 32, "revnet50": 224}
CLASSES = {"revnet18": 10, "revnet34": 1000, "revnet50": 1000}
CATS = ("total", "params", "optimizer", "shadows", "fifo", "workspace", "cmp_inputs", "cmp_stash")


def measure(a, inputs, stash):
    torch.cuda.set_device(0)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    H = IMAGE[a.model]
    units = PM.revnet(a.model, H, CLASSES[a.model])
    J = a.stages or len(units)
    counts = [1] * len(units) if J == len(units) else PM.partition(units, J, a.batch, H, H, 3)
    prec = L.BF16_TC if a.precision == "bf16" else L.FP32
    specs = PM.stage_specs(units, counts, a.batch, (H, H, 3), prec, 1e-4)
    for j, sp in enumerate(specs, 1):
        sp.compare_buffers = (L.CMP_INPUTS if inputs and j >= 2 else 0) | (L.CMP_STASH if stash else 0)
    free0, _ = torch.cuda.mem_get_info()
    pipe = Pipeline(specs, [0] * J, 0, 1, seed=1)
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((a.batch, H, H, 3), generator=gen, device="cuda")
    y = torch.randint(0, CLASSES[a.model], (a.batch,), generator=gen, device="cuda", dtype=torch.int32)
    loss = torch.zeros(1, device="cuda")
    ticks = a.ticks if a.ticks >= 0 else 2 * J
    for t in range(ticks):
        pipe.tick(t, True, x, y, 0.025, loss, report=False)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    tot = {k: 0 for k in CATS}
    per = []
    for j, s in sorted(pipe.stages.items()):
        m = s.memory()
        per.append({"stage": j, **{k: m[k] for k in CATS}})
        for k in CATS:
            tot[k] += m[k]
    # the paper excludes the first stage's input buffer: PETRA's own stage-1 FIFO holds
    # dataset inputs (the stem's), so it is left out of the comparable total as well
    s1_fifo = per[0]["fifo"]
    pipe.close()
    torch.cuda.synchronize()
    return {"input_buffer": inputs, "param_buffer": stash, "ticks": ticks, "J": J,
            "stage_bytes": tot, "stage_bytes_excl_stage1_fifo": tot["total"] - s1_fifo,
            "device_footprint_bytes": free0 - free1, "loss_finite": bool(torch.isfinite(loss).item()),
            "per_stage": per}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="revnet50")
    ap.add_argument("--stages", type=int, default=0, help="0: one stage per unit (= per residual block)")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--ticks", type=int, default=-1, help="-1: 2J (every ring slot written once)")
    a = ap.parse_args()
    GB = 1e9
    rows = [measure(a, i, s) for i, s in ((True, True), (True, False), (False, True), (False, False))]
    base = rows[0]["stage_bytes_excl_stage1_fifo"]
    table = []
    for r in rows:
        table.append({"input_buffer": r["input_buffer"], "param_buffer": r["param_buffer"],
                      "GB": round(r["stage_bytes_excl_stage1_fifo"] / GB, 2),
                      "saving_pct": round(100.0 * (1 - r["stage_bytes_excl_stage1_fifo"] / base), 1),
                      "device_footprint_GB": round(r["device_footprint_bytes"] / GB, 2),
                      "cmp_inputs_GB": round(r["stage_bytes"]["cmp_inputs"] / GB, 2),
                      "cmp_stash_GB": round(r["stage_bytes"]["cmp_stash"] / GB, 3)})
    print(json.dumps({"model": a.model, "batch": a.batch, "stages": rows[0]["J"], "precision": a.precision,
                      "method": "measured: real pipelines with the comparison buffers allocated and written every "
                                "tick (petra_stage_desc.compare_buffers); GB = sum of petra_stage_memory totals "
                                "(stage-1 FIFO excluded, as the paper excludes the first stage's buffer); "
                                "device_footprint = cudaMemGetInfo drop over the pipeline's life (mailboxes, "
                                "CUDA graphs and allocator granularity included)",
                      "paper_table3_GB": [44.5, 43.6, 21.2, 20.3], "paper_saving_pct": [0.0, 2.0, 52.3, 54.3],
                      "table": table, "runs": rows}))


if __name__ == "__main__":
    main()
