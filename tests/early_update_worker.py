"""Subprocess of tests/test_early_update_gpu.py: a RevNet-18 J=4 pipeline (the world-1 run of
tests/test_multirank_local_gpu.py) under the current PETRA_EARLY_UPDATE setting (read once per
process); losses and every stage's theta / v / running statistics saved to an .npz."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2406_02052_b200 import _lib as L  # noqa: E402
from tests.test_multirank_local_gpu import _run  # noqa: E402

precision = {"fp32": L.FP32, "bf16": L.BF16_TC}[sys.argv[1]]
losses, params, _ = _run(1, precision, True)
out = {f"loss_{k}": np.float32(v) for k, v in losses.items()}
for j, p in params.items():
    for i, a in enumerate(p if isinstance(p, (tuple, list)) else [p]):
        out[f"stage{j}_{i}"] = np.asarray(a)
np.savez(sys.argv[2], **out)
