"""Boundary items of SURVEY 8(b) (VERDICT r1 "next round" 8): the caller-installed
allocator and the non-finite latch on Delta."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.units import Branch, ConvBN, RevUnit  # noqa: E402
from paper_2406_02052_b200 import Stage, petra, _lib as L, models as PM  # noqa: E402
from tests.gpu_harness import oracle_to_product_units, pack_params, rand_params  # noqa: E402


def _stage(precision=L.BF16_TC, B=4):
    units = rand_params([RevUnit(0, Branch([ConvBN(64, 64, 3, 1)])), RevUnit(1, Branch([ConvBN(64, 64, 3, 1)]))], 3)
    st = Stage(PM.StageSpec(oracle_to_product_units(units), B, (8, 8, 64), precision), seed=0)
    th, bf = pack_params(units)
    st.set_params(th, np.zeros_like(th), bf)
    return st


_MB = [0]


def _tick(st, B=4, scale=1.0):
    mb = _MB[0]
    _MB[0] += 1
    g = torch.Generator(device="cuda").manual_seed(0)
    x = [torch.randn(B, 8, 8, 64, device="cuda", generator=g) for _ in range(2)]
    o = [torch.empty_like(x[0]) for _ in range(2)]
    st.forward(mb, x[0], x[1], o[0], o[1])
    d = [torch.randn(B, 8, 8, 64, device="cuda", generator=g) * scale for _ in range(2)]
    r = [torch.empty_like(x[0]) for _ in range(4)]
    st.backward(mb, o[0], o[1], d[0], d[1], *r, 0.01)
    torch.cuda.synchronize()


def test_torch_caching_allocator_holds_the_library_memory():
    torch.cuda.set_device(0)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    petra.use_torch_allocator(True)
    try:
        st = _stage()
        held = torch.cuda.memory_allocated() - base
        total = st.memory()["total"]
        assert held >= total > 0, (held, total)   # every byte the stage reports lives in torch's pool
        _tick(st)
        st.close()
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() == base  # all of it returned through release()
    finally:
        petra.use_torch_allocator(False)
    st = _stage()          # back on cudaMalloc: nothing in torch's pool
    assert torch.cuda.memory_allocated() == base
    st.close()


def test_nonfinite_delta_is_latched_and_reported():
    torch.cuda.set_device(0)
    st = _stage(L.FP32)
    _tick(st)
    st.get_params()                       # finite: no error
    _tick(st, scale=float("inf"))         # an infinite delta -> non-finite Delta
    with pytest.raises(L.PetraError) as e:
        st.get_params()
    assert e.value.name == "PETRA_E_NONFINITE" and "Delta" in str(e.value)
    st.close()
