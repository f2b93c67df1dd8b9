"""The TMA-staged BN passes (bn_apply / bn_bwd_reduce / bn_bwd_dz, DESIGN.md 7 "TMA-staged
BN passes") are bitwise identical to the register kernels they replace (advisor r1):
one stage tick per case with PETRA_BN_TMA_* = 1 (default) and = 0 in separate
processes, every output compared bit for bit.  Cases cover ragged chunks (M % Rc != 0),
many row blocks per channel tile, bf16 and fp32 z, the coupling addend, the stem's split
dy halves and a downsampling unit."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["stem_rev_ragged", "rev_pair_b64", "rev_pair_fp32_ragged", "ds_rev"]


def _run(case, tma, path):
    env = dict(os.environ)
    for k in ("PETRA_BN_TMA_APPLY", "PETRA_BN_TMA_REDUCE", "PETRA_BN_TMA_DZ"):
        env[k] = "1" if tma else "0"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "bn_tma_worker.py"), case, path], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return dict(np.load(path))


@pytest.mark.parametrize("case", CASES)
def test_bn_tma_bitwise_equals_register_kernels(case, tmp_path):
    a = _run(case, True, str(tmp_path / "tma.npz"))
    b = _run(case, False, str(tmp_path / "reg.npz"))
    assert sorted(a) == sorted(b)
    for k in a:
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k
