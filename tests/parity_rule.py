"""The GPU-vs-oracle comparison rule (SURVEY.md 8(c) "GPU-vs-oracle comparison
rule"; north_star tolerances; readings c22 and c25).

Per tensor T the test records
  rel_exact  = ||gpu - exact|| / ||exact||          (exact fp64 oracle)
  rel_bf16   = ||gpu - bf16|| / ||bf16||            (oracle under rules R1-R3, bf16 path only)
  floor      = ||bf16 - exact|| / ||exact||         (oracle vs oracle: what bf16 operands cost)
  max_el     = max |gpu - exact| / max |exact|
  outliers   = fraction of elements with |gpu - exact| > 1e-2 * rms(exact)

and passes it when
  fp32 path:  rel_exact <= 1e-4                                (north_star)
  bf16 path:  rel_bf16  <= 2e-2                                (north_star, vs the bf16 arithmetic)
              rel_exact <= 2e-2  if T is not mask-gated         (north_star, vs exact)
              rel_exact <= floor + 2e-2  if T is mask-gated     (reading c25)
"Mask-gated" tensors are the ones that carry a gradient through a ReLU mask (delta,
Delta, the momentum v): bf16 operands move ~0.1% of the mask decisions to the other
side of zero relative to exact arithmetic, and each flip passes or blocks an O(1)
gradient element, a floor (measured by `floor`, counted in flips by the test) that no
bf16-operand implementation can go under.  The same bf16 arithmetic with the exact
masks replayed stays within 2e-2 of exact on every tensor (tests/test_oracle_bf16.py
and the full-size test check that decomposition), so the floor is the flips alone.
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

    def add(self, name, got, exact, bf16=None, gated=False, tol=None):
        got = np.asarray(got, np.float64)
        exact = np.asarray(exact, np.float64)
        r_e = rel(got, exact)
        mx, out = elementwise(got, exact)
        row = {"name": name, "rel_exact": r_e, "max_el": mx, "outliers": out, "gated": bool(gated)}
        if self.bf16:
            if bf16 is None:
                raise ValueError(f"{name}: the bf16 path needs the bf16-rule oracle value")
            r_b = rel(got, bf16)
            fl = rel(bf16, exact)
            row.update(rel_bf16=r_b, floor=fl)
            t = TOL_BF16 if tol is None else tol
            ok = r_b <= t and (r_e <= fl + t if gated else r_e <= t)
        else:
            t = TOL_FP32 if tol is None else tol
            ok = r_e <= t
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
            s += f"  max_el {r['max_el']:.2e}  outliers {r['outliers']:.1e}" + ("  [gated]" if r["gated"] else "")
            lines.append(s)
        return "\n".join(lines)
