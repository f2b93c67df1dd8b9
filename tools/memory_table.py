"""Table 3 of the paper for this implementation: device memory of
RevNet-50 on ImageNet-shaped input, batch 64, one stage per residual block (J = 18,
PAPER.md:259), measured through petra_stage_memory, and the three buffered
configurations the paper compares against, derived from the same stages:

  input buffer  (delayed-gradient methods, PipeDream): every stage j >= 2 keeps the
                inputs of its 2(J-j)+1 in-flight micro-batches (PETRA: only its
                non-reversible units do); the first stage's buffer is excluded, as in
                the paper (its input is the dataset);
  param buffer  (weight stashing, PipeDream): 2(J-j) extra fp32 copies of theta_j.

Needs a GPU (allocates the 18 stages).  Prints one JSON object.
    python tools/memory_table.py [--model revnet50] [--stages 18] [--batch 64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2406_02052_b200 import Stage  # noqa: E402
from paper_2406_02052_b200 import _lib as L  # noqa: E402
from paper_2406_02052_b200 import models as PM  # noqa: E402

IMAGE = {"revnet18": 32, "revnet34": 32, "revnet50": 224}
CLASSES = {"revnet18": 10, "revnet34": 1000, "revnet50": 1000}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="revnet50")
    ap.add_argument("--stages", type=int, default=0, help="0: one stage per unit (= per residual block)")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    H = IMAGE[a.model]
    units = PM.revnet(a.model, H, CLASSES[a.model])
    J = a.stages or len(units)
    counts = [1] * len(units) if J == len(units) else PM.partition(units, J, a.batch, H, H, 3)
    prec = L.BF16_TC if a.precision == "bf16" else L.FP32
    specs = PM.stage_specs(units, counts, a.batch, (H, H, 3), prec)
    ins, _ = PM.shapes(units, a.batch, H, H, 3)
    GB = 1e9
    rows, i0 = [], 0
    tot = {k: 0 for k in ("total", "params", "optimizer", "shadows", "fifo", "workspace")}
    in_buf = par_buf = 0
    for j, spec in enumerate(specs, 1):
        st = Stage(spec, 0)
        m = st.memory()
        B, Hh, W, C = ins[i0]
        nonrev_first = units[i0].kind in (L.UNIT_STEM, L.UNIT_DS)
        in_bytes = (1 if units[i0].kind == L.UNIT_STEM else 2) * B * Hh * W * C * 4
        inflight = 2 * (J - j) + 1
        # input buffer of a delayed-gradient method: all in-flight inputs of stage j >= 2
        # (PETRA's own FIFO already holds them when the stage opens with a non-reversible unit)
        extra_in = 0 if j == 1 else inflight * in_bytes - (m["fifo"] if nonrev_first else 0)
        # first stage: its FIFO holds dataset inputs -- excluded as in the paper
        fifo_counted = 0 if j == 1 else m["fifo"]
        extra_par = 2 * (J - j) * st.n_params * 4
        for k in tot:
            tot[k] += m[k]
        tot["fifo"] -= m["fifo"] - fifo_counted
        tot["total"] -= m["fifo"] - fifo_counted
        in_buf += max(0, extra_in)
        par_buf += extra_par
        rows.append({"stage": j, "units": counts[j - 1], "memory": m, "input_buffer_extra": max(0, extra_in),
                     "param_buffer_extra": extra_par})
        st.close()
        i0 += counts[j - 1]
    petra = tot["total"]
    table = [
        {"input_buffer": True, "param_buffer": True, "GB": (petra + in_buf + par_buf) / GB},
        {"input_buffer": True, "param_buffer": False, "GB": (petra + in_buf) / GB},
        {"input_buffer": False, "param_buffer": True, "GB": (petra + par_buf) / GB},
        {"input_buffer": False, "param_buffer": False, "GB": petra / GB},
    ]
    base = table[0]["GB"]
    for r in table:
        r["saving_pct"] = round(100.0 * (1 - r["GB"] / base), 1)
        r["GB"] = round(r["GB"], 2)
    print(json.dumps({"model": a.model, "batch": a.batch, "stages": J, "precision": a.precision,
                      "paper_table3_GB": [44.5, 43.6, 21.2, 20.3], "paper_saving_pct": [0.0, 2.0, 52.3, 54.3],
                      "petra_measured_GB": {k: round(v / GB, 3) for k, v in tot.items()},
                      "table": table, "per_stage": rows}))


if __name__ == "__main__":
    main()
