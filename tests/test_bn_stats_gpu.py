"""Fused BN batch statistics at the benchmark's largest sizes (VERDICT r1 "next round" 5;
SURVEY 2.3 K1/K4; PAPER.md:259 batch statistics, reading c9).

The tensor-core convolutions compute the statistics of z (as stored, bf16: reading c24)
in their epilogue: per CTA the shifted sums of its valid rows, written as (count, mean,
M2), merged over CTAs with Chan's pairwise update in fp64 (petra_conv_bn_stats runs
exactly that path).  Against fp64 statistics of the very z the kernel stored, the mean
and the biased variance must agree to rel 1e-6 -- also when the channel means are
large against their spread (inputs offset by +4: E[z^2] - mean^2 would cancel ~1e3-fold)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2406_02052_b200 import _lib as L  # noqa: E402

# (name, geometry B, H, W, Ci, Co, k, s, engine): RevNet-50 / ImageNet b64 layer 1 (M = 200,704),
# its stem (M = 802,816), RevNet-18 / CIFAR b64 layer 1
GEOMS = {
    "r50_l1_1x1_256to64": ((64, 56, 56, 256, 64, 1, 1), 1),
    "r50_l1_3x3_64_halo": ((64, 56, 56, 64, 64, 3, 1), 2),
    "r50_l1_1x1_64to256": ((64, 56, 56, 64, 256, 1, 1), 1),
    "r50_stem_7x7s2": ((64, 224, 224, 3, 128, 7, 2), 1),
    "r18_l1_3x3_64_halo": ((64, 32, 32, 64, 64, 3, 1), 2),
    # cluster split-K plans (partials reduced through DSMEM, one statistics row per CTA)
    "r18_l3_3x3_256_cs": ((64, 8, 8, 256, 256, 3, 1), 1),
    "r18_l4_3x3_512_cs": ((64, 4, 4, 512, 512, 3, 1), 1),
    "r50_l4_3x3_512_cs": ((64, 7, 7, 512, 512, 3, 1), 1),
    "r50_l4_1x1_2048to512_cs": ((64, 7, 7, 2048, 512, 1, 1), 1),
}


@pytest.mark.parametrize("offset", [0.0, 4.0])
@pytest.mark.parametrize("case", sorted(GEOMS))
def test_fused_bn_stats_vs_fp64(case, offset):
    (B, H, W, Ci, Co, k, s), engine = GEOMS[case]
    g = L.PetraConvGeom(B, H, W, Ci, Co, k, s)
    rng = np.random.default_rng(7)
    x = (offset + rng.standard_normal((B, H, W, Ci))).astype(np.float32)
    # weights with a common positive part so that z's channel means are O(offset) or larger
    w = (rng.uniform(-1, 1, (Co, k, k, Ci)) * np.sqrt(3.0 / (k * k * Ci)) + 0.02).astype(np.float32)
    Ho, Wo = (H + 2 * ((k - 1) // 2) - k) // s + 1, (W + 2 * ((k - 1) // 2) - k) // s + 1
    z = np.empty((B * Ho * Wo, Co), np.float32)
    mean, var = np.empty(Co, np.float32), np.empty(Co, np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    L.call("petra_conv_bn_stats", C.byref(g), engine, p(x), p(w), p(z), p(mean), p(var))
    zd = z.astype(np.float64)
    m_ref = zd.mean(axis=0)
    v_ref = ((zd - m_ref) ** 2).mean(axis=0)
    sd = np.sqrt(v_ref)
    em = np.abs(mean - m_ref) / np.maximum(np.abs(m_ref), sd)
    ev = np.abs(var - v_ref) / v_ref
    ratio = float(np.median(np.abs(m_ref) / sd))
    print(f"{case} offset {offset}: |mean|/sd median {ratio:.1f}; mean rel err max {em.max():.2e}, "
          f"var rel err max {ev.max():.2e}")
    assert em.max() <= 1e-6, em.max()
    assert ev.max() <= 1e-6, ev.max()
