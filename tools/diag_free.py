"""Diagnostic: free-running standalone GPU stages (GPU messages, Python mailboxes)
vs the oracle tick engine, lr=0: isolates Pipeline bookkeeping from numerics."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import engine as E, models as OM
from tests.gpu_harness import nchw, nhwc, oracle_to_product_units, pack_like, pack_params, per_tensor_rel, rand_params, rel
from paper_2406_02052_b200 import Stage, models as PM

B, lr, n_mb, J = 4, float(sys.argv[1]) if len(sys.argv) > 1 else 0.0, 4, 4
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
reps, losses, grads = E.run_petra(ost, fn, n_mb, lr=lr, drain=True, record_grads=True)
gf = [None] * (J + 2); gb = [None] * (J + 2)
for r in reps:
    t = r.tick
    nf = [None] * (J + 2); nb = [None] * (J + 2)
    for j in range(1, J + 1):
        g = gst[j - 1]
        fmb, bmb = r.fwd_mb[j - 1], r.bwd_mb[j - 1]
        if j == 1 and fmb >= 0:
            xs, y = fn(fmb); fin = (fmb, [T(xs[0]), None], torch.tensor(y, dtype=torch.int32, device="cuda"))
        else:
            fin = gf[j]
        if j < J:
            if fmb >= 0:
                o = [torch.empty(g.out_shape, device="cuda") for _ in range(2)]
                g.forward(fmb, fin[1][0], fin[1][1], o[0], o[1]); nf[j + 1] = (fmb, o, fin[2])
            if bmb >= 0:
                m = gb[j]
                shp = (B,) + tuple(specs[j - 1].in_shape)
                res = [torch.empty(shp, device="cuda") for _ in range(4)] if j > 1 else [None] * 4
                keep = [x.clone() for x in m[1]]
                g.backward(bmb, *m[1], *res, lr)
                torch.cuda.synchronize()
                print("   inputs unchanged:", [torch.equal(a, b) for a, b in zip(keep, m[1])])
                if j > 1: nb[j - 1] = (bmb, res)
                torch.cuda.synchronize()
                errs = per_tensor_rel(groups[j - 1], g.get_grads(), pack_like(groups[j - 1], grads[(j, bmb)]))
                print(f"t{t} s{j} bwd mb{bmb}: grad max {max(e for _, e in errs):.1e}")
        elif fmb >= 0:
            shp = (B,) + tuple(specs[j - 1].in_shape)
            res = [torch.empty(shp, device="cuda") for _ in range(4)]
            loss = torch.zeros(1, device="cuda")
            g.tail(fmb, fin[1][0], fin[1][1], fin[2], lr, *res, loss)
            nb[j - 1] = (fmb, res)
            torch.cuda.synchronize()
            print(f"t{t} s{j} tail mb{fmb}: loss {loss.item():.6f} vs {losses[fmb]:.6f}",
                  "xt==in:", torch.equal(res[0], fin[1][0]), torch.equal(res[1], fin[1][1]))
    gf, gb = nf, nb
