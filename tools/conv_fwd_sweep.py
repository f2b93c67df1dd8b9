"""Forward-conv timing through petra_conv_bench: bf16 z with / without the fused BN
statistics, per R18/R50 geometry (device time per pass, CUDA events, no profiler)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2406_02052_b200 import _lib as L

GEOMS = [  # (B, H, W, Ci, Co, k, s)
    (64, 32, 32, 64, 64, 3, 1), (64, 16, 16, 128, 128, 3, 1), (64, 8, 8, 256, 256, 3, 1), (64, 4, 4, 512, 512, 3, 1),
    (64, 56, 56, 64, 256, 1, 1), (64, 56, 56, 256, 64, 1, 1), (64, 56, 56, 64, 64, 3, 1),
    (64, 28, 28, 512, 128, 1, 1), (64, 28, 28, 128, 512, 1, 1), (64, 28, 28, 128, 128, 3, 1),
    (64, 14, 14, 1024, 256, 1, 1), (64, 14, 14, 256, 1024, 1, 1), (64, 14, 14, 256, 256, 3, 1),
    (64, 7, 7, 2048, 512, 1, 1), (64, 7, 7, 512, 2048, 1, 1), (64, 7, 7, 512, 512, 3, 1),
    (64, 224, 224, 3, 128, 7, 2),
]
lib = L.lib()
for eng in (1, 2):
    for g in GEOMS:
        B, H, W, Ci, Co, k, s = g
        p = (k - 1) // 2
        Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
        flop = 2.0 * B * Ho * Wo * Co * k * k * Ci
        byt = 2.0 * (B * H * W * Ci + B * Ho * Wo * Co + Co * k * k * Ci)
        row = []
        for flags, nm in ((1, "z16"), (3, "z16+stats"), (0, "z32")):
            ms = C.c_float()
            st = lib.petra_conv_bench(0, eng, C.byref(L.PetraConvGeom(*g)), flags, 20, C.byref(ms))
            row.append(f"{nm}=" + (f"{ms.value * 1e3:7.1f}us {flop / ms.value / 1e9:6.1f}TF {byt / ms.value / 1e6:6.0f}GB/s"
                                   if st == 0 else f"n/a({st})"))
        print("eng", eng, g, " | ".join(row), flush=True)
