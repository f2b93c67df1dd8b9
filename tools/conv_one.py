"""One timed conv pass through petra_conv_bench (for ncu captures): argv = mode engine B H W Ci Co k s [flags]."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2406_02052_b200 import _lib as L

a = [int(v) for v in sys.argv[1:]]
mode, eng, geom = a[0], a[1], a[2:9]
flags = a[9] if len(a) > 9 else 0
ms = C.c_float()
st = L.lib().petra_conv_bench(mode, eng, C.byref(L.PetraConvGeom(*geom)), flags, 3, C.byref(ms))
print("status", st, "ms", ms.value)
