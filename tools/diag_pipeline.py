"""Diagnostic: per-tick, per-stage, per-tensor gradient error of the GPU
pipeline against the oracle tick engine (lr = 0)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import engine as E, models as OM
from tests.gpu_harness import nhwc, oracle_to_product_units, pack_like, pack_params, per_tensor_rel, rand_params
from paper_2406_02052_b200 import Pipeline, models as PM

B, lr, n_mb = 4, 0.0, 4
units = rand_params(OM.build_revnet("revnet18", 32, 10), 5)
counts = [5, 4, 4, 5]
groups = OM.group(units, counts)
init = [pack_params(g) for g in groups]
ost = [E.Stage(g, E.OptConfig()) for g in groups]
fn = lambda m: ([synth.images((B, 3, 32, 32), 0, m)], synth.labels(B, 10, 0, m))
pipe = Pipeline(PM.stage_specs(oracle_to_product_units(units), counts, B, (32, 32, 3)), seed=0)
for j, (th, bf) in enumerate(init, 1):
    pipe.stages[j].set_params(th, np.zeros_like(th), bf)
J = 4
for j, s in enumerate(ost, 1):
    s.j, s.J = j, J
fwd_box = [None] * (J + 2); bwd_box = [None] * (J + 2)
for t in range(n_mb + 2 * J - 2):
    # one oracle tick (same as run_petra)
    nf = [None] * (J + 2); nb = [None] * (J + 2); ran = {}
    for j, s in enumerate(ost, 1):
        s.lr = lr
        fin = E.Fwd(t, *fn(t)) if (j == 1 and t < n_mb) else (fwd_box[j] if j > 1 else None)
        if j < J:
            if fin is not None: nf[j + 1] = s.forward(fin)
            if bwd_box[j] is not None:
                out = s.backward(bwd_box[j]); ran[j] = bwd_box[j].mb
                if j > 1: nb[j - 1] = out
        elif fin is not None:
            _, out = s.tail_step(fin); ran[j] = fin.mb; nb[j - 1] = out
    fwd_box, bwd_box = nf, nb
    inject = t < n_mb
    x0 = lab = None
    if inject:
        xs, y = fn(t)
        x0 = torch.tensor(nhwc(xs[0]), dtype=torch.float32, device="cuda")
        lab = torch.tensor(y, dtype=torch.int32, device="cuda")
    pipe.tick(t, inject, x0, lab, lr, None)
    torch.cuda.synchronize()
    for j, mb in ran.items():
        errs = per_tensor_rel(groups[j - 1], pipe.stages[j].get_grads(), pack_like(groups[j - 1], ost[j - 1].last_grads))
        bad = [(n, f"{e:.1e}") for n, e in errs if e > 1e-5]
        print(f"tick {t} stage {j} mb {mb}: max {max(e for _, e in errs):.2e}", bad)
