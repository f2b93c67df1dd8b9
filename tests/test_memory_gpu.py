"""Table 3 accounting: petra_stage_memory
reports every device byte a stage allocated, by category; each category is
checked against its closed form from the stage's shapes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2406_02052_b200 import Stage  # noqa: E402
from paper_2406_02052_b200 import _lib as L  # noqa: E402
from paper_2406_02052_b200 import models as PM  # noqa: E402


def conv_weights(units):
    n = 0
    for u in units:
        for ci, co, k, s in list(u.layers) + list(u.proj):
            n += ci * co * k * k
    return n


@pytest.mark.parametrize("precision", [L.FP32, L.BF16_TC])
@pytest.mark.parametrize("k", [1, 2])
def test_stage_memory_categories(precision, k):
    torch.cuda.set_device(0)
    units = PM.revnet("revnet18")
    counts = [5, 4, 4, 5]
    specs = PM.stage_specs(units, counts, 8, (32, 32, 3), precision, accumulation_k=k)
    ins, _ = PM.shapes(units, 8, 32, 32, 3)
    i0 = 0
    for j, spec in enumerate(specs, 1):
        st = Stage(spec, 0)
        m = st.memory()
        us = units[i0:i0 + counts[j - 1]]
        assert m["params"] == 4 * (st.n_params + st.n_buffers)
        assert m["optimizer"] == 4 * st.n_params * (3 if k > 1 else 2)
        want_sh = 2 * 2 * conv_weights(us) if precision == L.BF16_TC else 0
        assert m["shadows"] == want_sh
        # FIFO: capacity 2(J-j)+1 (1 in the final stage) copies of each non-reversible unit's input
        cap = spec.fifo_capacity if j < len(specs) else 1
        fifo = 0
        tc = precision == L.BF16_TC
        for u, (B, H, W, C) in zip(us, ins[i0:i0 + counts[j - 1]]):
            # fp32 input (+ its bf16 conv operands on the tensor-core path: both DS halves;
            # the stem keeps only its 4-channel bf16 image copy there)
            if u.kind == L.UNIT_STEM:  # tensor cores: the 4-channel bf16 copy only (no fp32 kept)
                fifo += cap * B * H * W * (4 * 2 if tc else C * 4)
            elif u.kind == L.UNIT_DS:
                fifo += cap * 2 * B * H * W * C * (4 + (2 if tc else 0))
        assert m["fifo"] == fifo
        assert m["fifo_live"] == 0
        assert m["total"] == m["params"] + m["optimizer"] + m["shadows"] + m["fifo"] + m["workspace"]
        assert m["workspace"] > 0
        st.close()
        i0 += counts[j - 1]


def test_fifo_live_bytes_follow_pushes():
    """A forward pushes the input of every non-reversible unit; the backward pops it."""
    torch.cuda.set_device(0)
    units = PM.revnet("revnet18")
    spec = PM.stage_specs(units, [5, 4, 4, 5], 4, (32, 32, 3), L.FP32)[1]   # DS + REV units
    st = Stage(spec, 0)
    B, H, W, C = (4,) + tuple(spec.in_shape)
    x = [torch.randn(B, H, W, C, device="cuda") for _ in range(2)]
    o = [torch.empty(st.out_shape, device="cuda") for _ in range(2)]
    per = sum(2 * B * H * W * C * 4 for u in spec.units if u.kind == L.UNIT_DS)
    st.forward(0, x[0], x[1], o[0], o[1])
    st.forward(1, x[0], x[1], o[0], o[1])
    torch.cuda.synchronize()
    assert st.memory()["fifo_live"] == 2 * per
    d = [torch.randn_like(o[0]) for _ in range(2)]
    res = [torch.empty(B, H, W, C, device="cuda") for _ in range(4)]
    st.backward(0, o[0], o[1], d[0], d[1], *res, 0.0)
    torch.cuda.synchronize()
    assert st.memory()["fifo_live"] == per
    st.close()


def test_compare_buffers_measured_and_numerics_unchanged():
    """Table 3 comparison modes (petra_stage_desc.compare_buffers): the
    input ring holds fifo_capacity stage inputs (only for stages whose first unit is
    reversible: PETRA's own FIFO holds the others), the weight stash fifo_capacity - 1 =
    2(J-j) fp32 copies of theta; both are written every forward, and the trajectory stays
    PETRA's bitwise (theta, v and the losses equal the plain run's)."""
    import numpy as np
    from paper_2406_02052_b200 import Pipeline
    from paper_2406_02052_b200 import models as PM2
    torch.cuda.set_device(0)
    units = PM2.revnet("revnet18", 32, 10)
    counts = [5, 4, 4, 5]
    J, B = 4, 8
    out = {}
    for mode in (0, L.CMP_INPUTS | L.CMP_STASH):
        specs = PM2.stage_specs(units, counts, B, (32, 32, 3), L.BF16_TC)
        for sp in specs:
            sp.compare_buffers = mode
        pipe = Pipeline(specs, [0] * J, 0, 1, seed=3)
        gen = torch.Generator(device="cuda").manual_seed(0)
        loss = torch.zeros(1, device="cuda")
        losses = []
        for t in range(2 * J + 3):
            x = torch.randn((B, 32, 32, 3), generator=gen, device="cuda")
            y = torch.randint(0, 10, (B,), generator=gen, device="cuda", dtype=torch.int32)
            pipe.tick(t, True, x, y, 0.025, loss, report=False)
            torch.cuda.synchronize()
            losses.append(loss.item())
        mem = {j: s.memory() for j, s in pipe.stages.items()}
        prm = {j: s.get_params() for j, s in pipe.stages.items()}
        nparams = {j: s.n_params for j, s in pipe.stages.items()}
        pipe.close()
        out[mode] = (losses, prm, mem, nparams)
    l0, p0, m0, _ = out[0]
    l1, p1, m1, npar = out[L.CMP_INPUTS | L.CMP_STASH]
    assert l0 == l1
    for j in p0:
        for a, b in zip(p0[j], p1[j]):
            assert np.array_equal(a, b), j
    in_shapes = PM2.shapes(units, B, 32, 32, 3)[0]
    i0 = 0
    for j in range(1, J + 1):
        cap = 2 * (J - j) + 1
        first = units[i0]
        Bq, H, W, C = in_shapes[i0]
        exp_in = 0 if first.kind != L.UNIT_REV else cap * 2 * Bq * H * W * C * 4
        assert m1[j]["cmp_inputs"] == exp_in, j
        assert m1[j]["cmp_stash"] == (cap - 1) * npar[j] * 4, j
        assert m0[j]["cmp_inputs"] == 0 and m0[j]["cmp_stash"] == 0
        assert m1[j]["total"] - m0[j]["total"] == exp_in + (cap - 1) * npar[j] * 4, j
        i0 += counts[j - 1]
