"""Diagnostic: bf16 bottleneck/DS stage parity vs grid size / batch (padding vs numerics)."""
import sys
sys.path.insert(0, ".")
import tests.test_parity_gpu as T
from tests.gpu_harness import bf16_emulation
from paper_2406_02052_b200 import _lib as L

cases = {
    "ds_single_b3_14": (lambda: [T.ds_bott(128, 64, 256)], 3, [(3, 128, 14, 14)] * 2),
    "ds_single_b4_16": (lambda: [T.ds_bott(128, 64, 256)], 4, [(4, 128, 16, 16)] * 2),
    "ds_single_b2_32": (lambda: [T.ds_bott(128, 64, 256)], 2, [(2, 128, 32, 32)] * 2),
    "ds_basic_b4_16": (lambda: [T.ds_basic(128, 128)], 4, [(4, 128, 16, 16)] * 2),
    "bott_single_b4_16": (lambda: [T.bott(128, 64, 1)], 4, [(4, 128, 16, 16)] * 2),
    "two_conv_b4_16": (lambda: [T.RevUnit(1, T.Branch([T.ConvBN(128, 128, 3, 1), T.ConvBN(128, 128, 3, 1)]))],
                       4, [(4, 128, 16, 16)] * 2),
}
for name, c in cases.items():
    T.STAGE_CASES[name] = c
    try:
        with bf16_emulation():
            T._stage_tick(name, L.BF16_TC, None)
        print(name, "OK")
    except AssertionError as e:
        print(name, "FAIL", " | ".join(l.strip() for l in str(e).splitlines()[:-1]))
