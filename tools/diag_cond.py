"""Is the backward of stage 3 / mb 1 ill-conditioned w.r.t. x~ (oracle only)?"""
import sys, os, copy
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from oracle import engine as E, models as OM
from tests.gpu_harness import rand_params, rel

B, n_mb, J = 4, 4, 4
units = rand_params(OM.build_revnet("revnet18", 32, 10), 5)
groups = OM.group(units, [5, 4, 4, 5])
ost = [E.Stage(g, E.OptConfig()) for g in groups]
fn = lambda m: ([synth.images((B, 3, 32, 32), 0, m)], synth.labels(B, 10, 0, m))
for j, s in enumerate(ost, 1): s.j, s.J = j, J
fwd_box = [None] * (J + 2); bwd_box = [None] * (J + 2)
for t in range(5):
    nf = [None] * (J + 2); nb = [None] * (J + 2)
    for j, s in enumerate(ost, 1):
        s.lr = 0.0
        fin = E.Fwd(t, *fn(t)) if (j == 1 and t < n_mb) else (fwd_box[j] if j > 1 else None)
        if j < J:
            if fin is not None: nf[j + 1] = s.forward(fin)
            if bwd_box[j] is not None:
                out = s.backward(bwd_box[j])
                if j > 1: nb[j - 1] = out
        elif fin is not None:
            _, out = s.tail_step(fin); nb[j - 1] = out
    fwd_box, bwd_box = nf, nb
# at tick 5 stage 3 consumes bwd_box[3] (mb 1)
msg = bwd_box[3]
print("mb", msg.mb)
s3 = ost[2]
res = []
for mode in ["exact", "fp32", "fp32_again"]:
    st = copy.deepcopy(s3)
    m = copy.deepcopy(msg)
    if mode.startswith("fp32"):
        m.xs = [x.astype(np.float32).astype(np.float64) for x in m.xs]
        m.ds = [d.astype(np.float32).astype(np.float64) for d in m.ds]
    st.lr = 0.0
    out = st.backward(m)
    res.append((mode, st.last_grads, out))
for (n1, g1, o1), (n2, g2, o2) in [(res[0], res[1]), (res[1], res[2])]:
    print(n1, "vs", n2, "grad rel:", [f"{rel(a, b):.1e}" for a, b in zip(g1, g2)][:18])
# find small-variance BN channels in u2 recompute
st = copy.deepcopy(s3)
ys = msg.xs
for i in (3, 2):
    u = st.units[i]
    out, caches = u.phi.forward(ys[u.src])
    x, bc, mask = caches[0]
    print(f"unit {i}: min var {bc['var'].min():.3e} max invstd {bc['invstd'].max():.1f}; near-zero preact frac",
          np.mean(np.abs(u.phi.layers[0].gamma[None,:,None,None] * bc['xhat'] + u.phi.layers[0].beta[None,:,None,None]) < 1e-6))
    ys, _ = u.reconstruct(ys)
