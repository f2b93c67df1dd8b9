"""Cluster split-K A/B per layer: forward (bf16 z + fused statistics) and dgrad device time
through petra_conv_bench for the few-tile layers, under the current PETRA_CONV_CS setting."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
from paper_2406_02052_b200 import _lib as L

GEOMS = [(64, 8, 8, 256, 256, 3, 1), (64, 4, 4, 512, 512, 3, 1), (64, 7, 7, 512, 512, 3, 1),
         (64, 7, 7, 2048, 512, 1, 1), (64, 8, 8, 128, 256, 3, 2), (64, 4, 4, 256, 512, 3, 2)]
lib = L.lib()
tag = os.environ.get("PETRA_CONV_CS", "1") + "/" + os.environ.get("PETRA_CONV_CS_CTAS", "128")
for g in GEOMS:
    B, H, W, Ci, Co, k, s = g
    p = (k - 1) // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    flop = 2.0 * B * Ho * Wo * Co * k * k * Ci
    plan = (C.c_int32 * 3)()
    lib.petra_conv_plan(C.byref(L.PetraConvGeom(*g)), 0, plan)
    row = []
    for mode, flags, nm in ((0, 3, "fwd"), (1, 0, "dgrad")):
        ms = C.c_float()
        st = lib.petra_conv_bench(mode, 1, C.byref(L.PetraConvGeom(*g)), flags, 50, C.byref(ms))
        row.append(f"{nm}=" + (f"{ms.value * 1e3:7.1f}us {flop / ms.value / 1e9:6.1f}TF" if st == 0 else f"n/a({st})"))
    print(f"CS {tag} {g} plan {tuple(plan)} " + " | ".join(row), flush=True)
