"""Kernel-level GPU tests (T1): one convolution pass through petra_conv_run.
  * SIMT fp32 kernels vs the oracle's fp64 conv / VJP (rel 1e-6);
  * tcgen05 bf16 kernels vs the SIMT kernels on bf16-exact inputs: every product
    is exact in fp32 on both, so only the summation order differs (rel 1e-5)."""
import ctypes as C
import os

import numpy as np
import pytest

import synth
from oracle import primitives as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
from paper_2406_02052_b200 import _lib as L  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16_exact(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).to(torch.float32).numpy()


def conv_run(mode, engine, geom, a, b, addend=None):
    B, H, W, Ci, Co, k, s = geom
    g = L.PetraConvGeom(B, H, W, Ci, Co, k, s)
    p = (k - 1) // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    n_out = {0: B * Ho * Wo * Co, 1: B * H * W * Ci, 2: Co * k * k * Ci}[mode]
    out = np.zeros(n_out, np.float32)
    a, b = np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32)
    ad = None if addend is None else np.ascontiguousarray(addend, np.float32)
    st = L.lib().petra_conv_run(mode, engine, C.byref(g), a.ctypes.data, b.ctypes.data,
                                None if ad is None else ad.ctypes.data, out.ctypes.data)
    if st != 0:
        raise L.PetraError(st, "petra_conv_run", "")
    return out


GEOMS = [  # (B, H, W, Ci, Co, k, stride)
    (2, 32, 32, 64, 64, 3, 1), (2, 16, 16, 128, 128, 3, 1), (8, 8, 8, 256, 256, 3, 1),
    (8, 4, 4, 512, 512, 3, 1), (2, 16, 16, 256, 64, 1, 1), (2, 16, 16, 64, 256, 1, 1),
    (4, 8, 8, 64, 192, 3, 1),
    # stride-2 downsampling convs (R18 DS units: 3x3/s2 Phi_s, 1x1/s2 projections)
    (2, 32, 32, 64, 128, 3, 2), (2, 32, 32, 64, 128, 1, 2), (8, 16, 16, 128, 256, 3, 2),
    (8, 8, 8, 256, 512, 3, 2), (8, 8, 8, 256, 512, 1, 2),
    # ImageNet / ResNet-50 grids (56, 28, 14, 7): padded tiles (Wb = 64, 32, 16, 8), masked rows
    (2, 56, 56, 64, 64, 3, 1), (2, 56, 56, 64, 256, 1, 1), (2, 28, 28, 128, 128, 3, 1),
    (2, 14, 14, 256, 256, 3, 1), (3, 7, 7, 512, 512, 3, 1), (2, 56, 56, 64, 128, 3, 2),
    (2, 28, 28, 128, 256, 1, 2), (3, 14, 14, 256, 512, 3, 2), (1, 12, 20, 64, 64, 3, 1),
    (2, 14, 14, 128, 64, 1, 1), (2, 14, 14, 64, 64, 3, 1), (2, 14, 14, 64, 128, 1, 1),
]
# the benchmark's few-tile, long-K layers at b64 (cluster split-K plans): R18 layers 3, 4;
# R50 layer 4 (7x7 grid: masked padding rows) 3x3 and 1x1
CS_GEOMS = [(64, 8, 8, 256, 256, 3, 1), (64, 4, 4, 512, 512, 3, 1), (64, 7, 7, 512, 512, 3, 1),
            (64, 7, 7, 2048, 512, 1, 1)]
GEOMS += CS_GEOMS
SIMT_GEOMS = GEOMS[:2] + [(2, 9, 7, 3, 16, 3, 1), (2, 10, 10, 16, 32, 3, 2), (2, 9, 9, 8, 12, 1, 2),
                          (2, 15, 15, 3, 8, 7, 2)]


def inputs(geom, seed):
    B, H, W, Ci, Co, k, s = geom
    p = (k - 1) // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    x = bf16_exact(synth.normal((B, H, W, Ci), seed, 1))
    w = bf16_exact(synth.normal((Co, k, k, Ci), seed, 2) / np.sqrt(k * k * Ci))
    dz = bf16_exact(synth.normal((B, Ho, Wo, Co), seed, 3))
    add = synth.normal((B, H, W, Ci), seed, 4).astype(np.float32)
    return x, w, dz, add


@pytest.mark.parametrize("geom", SIMT_GEOMS)
def test_simt_conv_vs_oracle(geom):
    B, H, W, Ci, Co, k, s = geom
    x, w, dz, add = inputs(geom, 1)
    xo, wo, dzo = x.transpose(0, 3, 1, 2), w.transpose(0, 3, 1, 2), dz.transpose(0, 3, 1, 2)
    want_z = P.conv2d(xo.astype(np.float64), wo.astype(np.float64), s, (k - 1) // 2)
    dx_w, dw_w = P.conv2d_vjp(xo.astype(np.float64), wo.astype(np.float64), s, (k - 1) // 2, dzo.astype(np.float64))
    z = conv_run(0, 0, geom, x, w).reshape(want_z.transpose(0, 2, 3, 1).shape)
    assert rel(z, want_z.transpose(0, 2, 3, 1)) < 1e-6
    dx = conv_run(1, 0, geom, dz, w, add).reshape(add.shape)
    assert rel(dx, dx_w.transpose(0, 2, 3, 1) + add) < 1e-6
    dw = conv_run(2, 0, geom, dz, x).reshape(w.shape)
    assert rel(dw, dw_w.transpose(0, 2, 3, 1)) < 1e-6


@pytest.mark.parametrize("geom", GEOMS)
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_tc_conv_vs_simt(geom, mode):
    x, w, dz, add = inputs(geom, 2)
    a = x if mode == 0 else dz
    b = x if mode == 2 else w
    addend = add if mode == 1 else None
    assert L.lib().petra_conv_engine(C.byref(L.PetraConvGeom(*geom)), mode, L.BF16_TC) == 1
    ref = conv_run(mode, 0, geom, a, b, addend)
    got = conv_run(mode, 1, geom, a, b, addend)
    assert rel(got, ref) < 1e-5, rel(got, ref)


# stems: <= 4 input channels -> the gathered-im2col tensor-core kernels (forward, wgrad)
STEM_GEOMS = [(4, 32, 32, 3, 64, 3, 1), (2, 30, 30, 3, 64, 7, 2), (3, 17, 19, 3, 128, 7, 2),
              (1, 224, 224, 3, 64, 7, 2), (2, 12, 12, 4, 256, 5, 1), (2, 16, 16, 1, 64, 3, 1),
              (2, 9, 11, 2, 128, 1, 1)]


@pytest.mark.parametrize("geom", STEM_GEOMS)
@pytest.mark.parametrize("mode", [0, 2])
def test_stem_tc_vs_simt(geom, mode):
    x, w, dz, _ = inputs(geom, 5)
    a = x if mode == 0 else dz
    b = w if mode == 0 else x
    assert L.lib().petra_conv_engine(C.byref(L.PetraConvGeom(*geom)), mode, L.BF16_TC) == 1
    assert L.lib().petra_conv_engine(C.byref(L.PetraConvGeom(*geom)), 1, L.BF16_TC) == 0  # no stem dgrad
    ref = conv_run(mode, 0, geom, a, b)
    got = conv_run(mode, 1, geom, a, b)
    assert rel(got, ref) < 1e-5, rel(got, ref)


# zero-bordered operands (engine 2): 3x3 stride-1 grids large enough for the halo
# kernel (>= 3/4 of a wave of 128-row tiles), plus small / strided ones that read the
# padded buffers through interior TMA views
PAD_GEOMS = [(16, 32, 32, 64, 64, 3, 1), (8, 56, 56, 64, 64, 3, 1), (16, 16, 16, 128, 128, 3, 1),
             (64, 8, 8, 256, 256, 3, 1), (4, 28, 28, 128, 256, 3, 1), (2, 16, 16, 64, 64, 3, 1),
             (3, 14, 14, 256, 128, 3, 1)]


@pytest.mark.parametrize("geom", PAD_GEOMS)
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_tc_padded_operands_vs_simt(geom, mode):
    x, w, dz, add = inputs(geom, 7)
    a = x if mode == 0 else dz
    b = x if mode == 2 else w
    addend = add if mode == 1 else None
    ref = conv_run(mode, 0, geom, a, b, addend)
    got = conv_run(mode, 2, geom, a, b, addend)
    assert rel(got, ref) < 1e-5, rel(got, ref)


@pytest.mark.parametrize("geom,mode", [(g, m) for g in CS_GEOMS for m in (0, 1) if not (g[3] == 2048 and m == 1)])
@pytest.mark.skipif(os.environ.get("PETRA_CONV_CS", "0") != "1" and os.environ.get("PETRA_CONV_PAIR", "0") != "1",
                    reason="default plans (tests/test_conv_modes_gpu.py sets the modes)")
def test_conv_mode_plan(geom, mode):
    """Under PETRA_CONV_CS=1 the few-tile layers take the cluster split-K plan; under
    PETRA_CONV_PAIR=1 every N >= 128 tile runs on CTA pairs (plan[2] == -2)."""
    plan = (C.c_int32 * 3)()
    L.call("petra_conv_plan", C.byref(L.PetraConvGeom(*geom)), mode, plan)
    BN, splits, cs = plan
    if os.environ.get("PETRA_CONV_CS", "0") == "1":
        assert cs in (2, 4) and splits == cs, tuple(plan)
    else:
        assert (cs == -2) == (BN >= 128) and splits == 1, tuple(plan)
