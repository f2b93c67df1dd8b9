"""Diagnostic: drive standalone GPU stages with the ORACLE's messages at every
tick (state injection, lr=0) and compare each stage's outputs and gradients."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import engine as E, models as OM
from tests.gpu_harness import nchw, nhwc, oracle_to_product_units, pack_like, pack_params, per_tensor_rel, rand_params, rel
from paper_2406_02052_b200 import Stage, models as PM

B, lr, n_mb, J = 4, 0.0, 4, 4
units = rand_params(OM.build_revnet("revnet18", 32, 10), 5)
counts = [5, 4, 4, 5]
groups = OM.group(units, counts)
init = [pack_params(g) for g in groups]
ost = [E.Stage(g, E.OptConfig()) for g in groups]
specs = PM.stage_specs(oracle_to_product_units(units), counts, B, (32, 32, 3))
gst = [Stage(s, 0) for s in specs]
for s, (th, bf) in zip(gst, init):
    s.set_params(th, np.zeros_like(th), bf)
fn = lambda m: ([synth.images((B, 3, 32, 32), 0, m)], synth.labels(B, 10, 0, m))
T = lambda a: torch.tensor(nhwc(a), dtype=torch.float32, device="cuda")
for j, s in enumerate(ost, 1):
    s.j, s.J = j, J
fwd_box = [None] * (J + 2); bwd_box = [None] * (J + 2)
for t in range(n_mb + 2 * J - 2):
    nf = [None] * (J + 2); nb = [None] * (J + 2)
    for j, s in enumerate(ost, 1):
        s.lr = lr
        g = gst[j - 1]
        fin = E.Fwd(t, *fn(t)) if (j == 1 and t < n_mb) else (fwd_box[j] if j > 1 else None)
        if j < J:
            if fin is not None:
                out = s.forward(fin); nf[j + 1] = out
                o = [torch.empty(g.out_shape, device="cuda") for _ in range(2)]
                g.forward(fin.mb, T(fin.xs[0]), T(fin.xs[1]) if len(fin.xs) > 1 else None, o[0], o[1])
                torch.cuda.synchronize()
                e = max(rel(nchw(o[h].cpu().numpy()), out.xs[h]) for h in range(2))
                print(f"t{t} s{j} fwd mb{fin.mb}: {e:.1e}")
            bm = bwd_box[j]
            if bm is not None:
                out = s.backward(bm)
                if j > 1: nb[j - 1] = out
                ins = gst[j - 1]
                shp = (B,) + tuple(specs[j - 1].in_shape)
                res = [torch.empty(shp, device="cuda") for _ in range(4)] if j > 1 else [None] * 4
                g.backward(bm.mb, T(bm.xs[0]), T(bm.xs[1]), T(bm.ds[0]), T(bm.ds[1]), *res, lr)
                torch.cuda.synchronize()
                errs = per_tensor_rel(groups[j - 1], g.get_grads(), pack_like(groups[j - 1], s.last_grads))
                eo = [rel(nchw(res[k].cpu().numpy()), (out.xs + out.ds)[k]) for k in range(4)] if j > 1 else []
                print(f"t{t} s{j} bwd mb{bm.mb}: grad max {max(e for _, e in errs):.1e} outs " + " ".join(f"{x:.1e}" for x in eo),
                      [(n, f"{e:.1e}") for n, e in errs if e > 1e-5])
        elif fin is not None:
            loss, out = s.tail_step(fin); nb[j - 1] = out
    fwd_box, bwd_box = nf, nb
