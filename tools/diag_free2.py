"""Oracle and GPU stages in lockstep; at each backward also run a COPY of the
oracle stage on the GPU's own message, to see whether the GPU message or the
GPU backward is at fault."""
import sys, os, copy
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
H = lambda t: nchw(t.cpu().numpy().astype(np.float64))
for j, s in enumerate(ost, 1): s.j, s.J = j, J
of = [None] * (J + 2); ob = [None] * (J + 2)
gf = [None] * (J + 2); gb = [None] * (J + 2)
for t in range(n_mb + 2 * J - 2):
    nof = [None] * (J + 2); nob = [None] * (J + 2); ngf = [None] * (J + 2); ngb = [None] * (J + 2)
    for j in range(1, J + 1):
        s, g = ost[j - 1], gst[j - 1]
        s.lr = lr
        if j == 1:
            fin = E.Fwd(t, *fn(t)) if t < n_mb else None
            gfin = (t, [T(fin.xs[0]), None], torch.tensor(fin.labels, dtype=torch.int32, device="cuda")) if fin else None
        else:
            fin, gfin = of[j], gf[j]
        if j < J:
            if fin is not None:
                nof[j + 1] = s.forward(fin)
                o = [torch.empty(g.out_shape, device="cuda") for _ in range(2)]
                g.forward(gfin[0], gfin[1][0], gfin[1][1], o[0], o[1]); ngf[j + 1] = (gfin[0], o, gfin[2])
            if ob[j] is not None:
                msg, gm = ob[j], gb[j]
                # oracle copy on the GPU's message
                sc = copy.deepcopy(s)
                gmsg = E.Bwd(msg.mb, [H(gm[1][0]), H(gm[1][1])], [H(gm[1][2]), H(gm[1][3])])
                sc.backward(gmsg)
                out = s.backward(msg)
                if j > 1: nob[j - 1] = out
                shp = (B,) + tuple(specs[j - 1].in_shape)
                res = [torch.empty(shp, device="cuda") for _ in range(4)] if j > 1 else [None] * 4
                g.backward(msg.mb, *gm[1], *res, lr)
                if j > 1: ngb[j - 1] = (msg.mb, res)
                torch.cuda.synchronize()
                gg = g.get_grads()
                e_gpu_vs_orc = max(e for _, e in per_tensor_rel(groups[j - 1], gg, pack_like(groups[j - 1], s.last_grads)))
                e_gpu_vs_orcgpumsg = max(e for _, e in per_tensor_rel(groups[j - 1], gg, pack_like(groups[j - 1], sc.last_grads)))
                e_msgs = [rel(H(a), b) for a, b in zip(gm[1], msg.xs + msg.ds)]
                print(f"t{t} s{j} mb{msg.mb}: gpu-vs-oracle {e_gpu_vs_orc:.1e}  gpu-vs-oracle(gpu msg) {e_gpu_vs_orcgpumsg:.1e}  msg err " + " ".join(f"{e:.1e}" for e in e_msgs))
        elif fin is not None:
            _, out = s.tail_step(fin); nob[j - 1] = out
            shp = (B,) + tuple(specs[j - 1].in_shape)
            res = [torch.empty(shp, device="cuda") for _ in range(4)]
            loss = torch.zeros(1, device="cuda")
            g.tail(gfin[0], gfin[1][0], gfin[1][1], gfin[2], lr, *res, loss)
            ngb[j - 1] = (gfin[0], res)
    of, ob, gf, gb = nof, nob, ngf, ngb
