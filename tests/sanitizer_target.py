"""Small-shape workload for tests/test_sanitizer_gpu.py (run under compute-sanitizer):
the tcgen05 / TMEM / TMA convolution kernels (conv_tc forward / dgrad / wgrad, the halo
forward / dgrad / wgrad, the stem), the fused BN statistics, and one bf16 stage tick
(TMA-staged BN apply / backward-reduce / dz, the update, the max-pool stem, the evaluation
forward) through the C ABI."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_02052_b200 import _lib as L  # noqa: E402


def conv(mode, engine, geom):
    B, H, W, Ci, Co, k, s = geom
    g = L.PetraConvGeom(*geom)
    Ho, Wo = (H + 2 * ((k - 1) // 2) - k) // s + 1, (W + 2 * ((k - 1) // 2) - k) // s + 1
    r = np.random.default_rng(0)
    nx, nz, nw = B * H * W * Ci, B * Ho * Wo * Co, Co * k * k * Ci
    a = r.standard_normal(nx if mode == 0 else nz).astype(np.float32)
    b = r.standard_normal(nx if mode == 2 else nw).astype(np.float32)
    out = np.empty(nz if mode == 0 else (nx if mode == 1 else nw), np.float32)
    p = lambda x: x.ctypes.data_as(C.c_void_p)
    L.call("petra_conv_run", mode, engine, C.byref(g), p(a), p(b), None, p(out))


def main():
    torch.cuda.set_device(0)
    for mode in (0, 1, 2):
        conv(mode, 1, (2, 8, 8, 64, 128, 3, 1))      # conv_tc (implicit im2col, 3x3)
        conv(mode, 1, (2, 8, 8, 64, 64, 3, 2))       # stride 2 (dgrad: four phases)
        conv(mode, 2, (4, 16, 16, 64, 64, 3, 1))     # halo kernels (zero-bordered operands)
    conv(0, 1, (2, 16, 16, 3, 64, 3, 1))             # stem (gathered im2col)
    conv(2, 1, (2, 16, 16, 3, 64, 3, 1))
    g = L.PetraConvGeom(4, 16, 16, 64, 64, 3, 1)
    x = np.random.default_rng(1).standard_normal(4 * 16 * 16 * 64).astype(np.float32)
    w = np.random.default_rng(2).standard_normal(64 * 9 * 64).astype(np.float32) * 0.05
    z = np.empty(4 * 16 * 16 * 64, np.float32)
    m, v = np.empty(64, np.float32), np.empty(64, np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    L.call("petra_conv_bn_stats", C.byref(g), 2, p(x), p(w), p(z), p(m), p(v))
    # one bf16 stage tick: stem + reversible pair + DS (TMA-staged BN passes, update)
    sys.argv = [sys.argv[0]]
    from tests import bn_tma_worker as W
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        W.main("stem_rev_ragged", os.path.join(d, "a.npz"))
        W.main("ds_rev", os.path.join(d, "b.npz"))
        W.main("stem_maxpool", os.path.join(d, "c.npz"))
    torch.cuda.synchronize()
    print("sanitizer target done")


if __name__ == "__main__":
    main()
