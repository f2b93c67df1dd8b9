"""Kernel-level timing sweep through petra_conv_bench (device time per pass, CUDA
events; no profiler).  Prints achieved TFLOP/s per engine for the R18/R50 geometries."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2406_02052_b200 import _lib as L

GEOMS = [  # (B, H, W, Ci, Co, k, s)
    (64, 32, 32, 64, 64, 3, 1), (64, 16, 16, 128, 128, 3, 1), (64, 8, 8, 256, 256, 3, 1), (64, 4, 4, 512, 512, 3, 1),
    (64, 56, 56, 64, 64, 3, 1), (64, 56, 56, 64, 256, 1, 1), (64, 56, 56, 256, 64, 1, 1),
    (64, 28, 28, 128, 128, 3, 1), (64, 14, 14, 256, 256, 3, 1), (64, 7, 7, 512, 512, 3, 1),
    (64, 32, 32, 64, 128, 3, 2), (64, 224, 224, 3, 64, 7, 2),
]
ENG = {0: "simt", 1: "tc", 2: "tc_pad"}
lib = L.lib()
for g in GEOMS:
    B, H, W, Ci, Co, k, s = g
    p = (k - 1) // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    flop = 2.0 * B * Ho * Wo * Co * k * k * Ci
    row = []
    for mode in (0, 1, 2):
        for eng in (1, 2):
            ms = C.c_float()
            st = lib.petra_conv_bench(mode, eng, C.byref(L.PetraConvGeom(*g)), 1 if mode == 0 else 0, 20,
                                      C.byref(ms))
            row.append(f"{'fdw'[mode]}:{ENG[eng]}=" + (f"{ms.value * 1e3:7.1f}us/{flop / ms.value / 1e9:6.1f}TF"
                                                       if st == 0 else f"n/a({st})"))
    print(g, " ".join(row), flush=True)
