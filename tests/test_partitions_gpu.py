"""Every contiguous stage grouping the partitioner can produce runs: for J = 1 .. #units
the Pipeline (C++ planning of output / reconstruction buffers, FIFOs, mailboxes) of
RevNet-18 and RevNet-50 (small images, batch 2, bf16 tensor-core path and fp32) is
built and driven through fill, steady state and drain.  Integer reports follow the
closed forms of Table 1 (forward at t = m + j - 1, backward at
t = m + 2J - j - 1) and every loss is finite.  (The RevNet-50 J=4 grouping once
put a reversible unit before a downsampling unit in the final stage and failed.)"""
import math

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2406_02052_b200 import Pipeline  # noqa: E402
from paper_2406_02052_b200 import _lib as L  # noqa: E402
from paper_2406_02052_b200 import models as PM  # noqa: E402


@pytest.mark.parametrize("model,H", [("revnet18", 32), ("revnet50", 64)])
@pytest.mark.parametrize("precision", [L.BF16_TC, L.FP32])
def test_every_partition_runs(model, H, precision):
    torch.cuda.set_device(0)
    units = PM.revnet(model, H, 10)
    n = len(units)
    B, T = 2, 3
    for J in range(1, n + 1):
        counts = PM.partition(units, J, B, H, H, 3)
        specs = PM.stage_specs(units, counts, B, (H, H, 3), precision)
        pipe = Pipeline(specs, seed=J)
        loss = torch.zeros(1, device="cuda")
        for t in range(T + 2 * J - 2):
            inject = t < T
            x = torch.randn(B, H, H, 3, device="cuda") if inject else None
            y = torch.randint(0, 10, (B,), device="cuda", dtype=torch.int32) if inject else None
            r = pipe.tick(t, inject, x, y, 0.01, loss)
            for j in range(1, J + 1):
                m_f = t - (j - 1)
                assert r["fwd_mb"][j - 1] == (m_f if 0 <= m_f < T else -1), (J, t, j, r)
                m_b = t - (2 * J - j - 1)
                assert r["bwd_mb"][j - 1] == (m_b if 0 <= m_b < T else -1), (J, t, j, r)
            if r["fwd_mb"][-1] >= 0:
                torch.cuda.synchronize()
                assert math.isfinite(loss.item()), (J, t)
        torch.cuda.synchronize()
        pipe.close()
