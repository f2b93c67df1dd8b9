"""The GPU-vs-oracle comparison rule (SURVEY.md 8(c) "GPU-vs-oracle comparison
rule"; north_star tolerances; readings c22 and c25).

Per tensor T the test records
  rel_exact  = ||gpu - exact|| / ||exact||          (exact fp64 oracle)
  rel_bf16   = ||gpu - bf16|| / ||bf16||            (oracle under rules R1-R3, bf16 path only)
  floor      = ||bf16 - exact|| / ||exact||         (oracle vs oracle: what bf16 operands cost)
  order      = max over alternatives A of ||A - ref|| / ||ref||   (oracle vs oracle: what
               another rounding costs; ref = exact for fp32, bf16 for bf16), A =
                 ref_acc32: the same oracle with its convolutions accumulated and its stored
                            tensors rounded in fp32 (oracle.primitives.fp32_accumulation) --
                            a sampled alternative rounding;
                 ref_band:  the same oracle with every mask decision whose pre-activation
                            lies within the fp32 rounding band (2e-5 rms, 4 sigma of a
                            4608-term fp32 dot product) of zero taken the other way -- a
                            deterministic upper estimate when the sample flips nothing
  max_el     = max |gpu - exact| / max |exact|
  outliers   = fraction of elements with |gpu - exact| > 1e-2 * rms(exact)

and passes it when (t = 1e-4 fp32, 2e-2 bf16: north_star)
  T not mask-gated:  fp32  rel_exact <= t
                     bf16  rel_bf16 <= t  and  rel_exact <= t
  T mask-gated:      fp32  rel_exact <= t + 2 * order                      (reading c25)
                     bf16  rel_bf16  <= t + 2 * order
                           rel_exact <= t + floor + 2 * order
"Mask-gated" tensors carry a gradient through a ReLU mask: delta, Delta, the momentum
v and theta after the update (theta^{t+1} = theta^t - lr (Delta + ...)).  A mask is an
integer decided from floating point: an implementation that rounds differently moves
the decisions whose pre-activation lies within its rounding difference of zero, and
each flipped decision passes or blocks an O(1) gradient element.  bf16 operands move
~0.1% of the decisions relative to exact arithmetic (counted by the tests): `floor`,
which no bf16-operand implementation can go under -- the same bf16 arithmetic with the
exact masks replayed stays within 2e-2 of exact on every tensor (tests/test_oracle_bf16.py
and the full-size test check that decomposition).  A different summation order of the
same arithmetic moves far fewer (counted): `order`, measured on the oracle itself; the
GPU's fp32 accumulation is such a rounding, and the factor 2 covers the statistical
spread between two draws of the same process.  Tensors computed before any mask decision
(forward outputs, x~, running statistics, the loss) get no allowance.
"""
from __future__ import annotations

import numpy as np

from tests.gpu_harness import elementwise, rel

TOL_FP32 = 1e-4
TOL_BF16 = 2e-2


class Report:
    def __init__(self, precision_bf16: bool):
        self.bf16 = precision_bf16
        self.rows = []

    def add(self, name, got, exact, bf16=None, gated=False, tol=None, alt=None):
        """alt: the alternatives' values of T (a list: ref_acc32, ref_band), the `order`
        measurement; required for mask-gated tensors."""
        got = np.asarray(got, np.float64)
        exact = np.asarray(exact, np.float64)
        r_e = rel(got, exact)
        mx, out = elementwise(got, exact)
        row = {"name": name, "rel_exact": r_e, "max_el": mx, "outliers": out, "gated": bool(gated)}
        if gated and alt is None:
            raise ValueError(f"{name}: a mask-gated tensor needs the fp32-accumulation oracle value")
        ref = bf16 if self.bf16 else exact
        if gated and not isinstance(alt, (list, tuple)):
            alt = [alt]
        order = max(rel(a, ref) for a in alt) if gated else 0.0
        row["order"] = order
        if self.bf16:
            if bf16 is None:
                raise ValueError(f"{name}: the bf16 path needs the bf16-rule oracle value")
            r_b = rel(got, bf16)
            fl = rel(bf16, exact)
            row.update(rel_bf16=r_b, floor=fl)
            t = TOL_BF16 if tol is None else tol
            ok = r_b <= t + 2 * order and r_e <= t + (fl if gated else 0.0) + 2 * order
        else:
            t = TOL_FP32 if tol is None else tol
            ok = r_e <= t + 2 * order
        row["ok"] = bool(ok)
        self.rows.append(row)
        return ok

    @property
    def ok(self):
        return all(r["ok"] for r in self.rows)

    def worst(self, key):
        vals = [r[key] for r in self.rows if key in r]
        return max(vals) if vals else 0.0

    def text(self):
        lines = []
        for r in self.rows:
            s = f"{'ok ' if r['ok'] else 'BAD'} {r['name']:28s} exact {r['rel_exact']:.2e}"
            if "rel_bf16" in r:
                s += f"  bf16 {r['rel_bf16']:.2e}  floor {r['floor']:.2e}"
            if r["gated"]:
                s += f"  order {r['order']:.2e}"
            s += f"  max_el {r['max_el']:.2e}  outliers {r['outliers']:.1e}" + ("  [gated]" if r["gated"] else "")
            lines.append(s)
        return "\n".join(lines)
