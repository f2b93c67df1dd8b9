"""Pins of the oracle's bf16 mode (readings c22 and c25), CPU only.

* ``bf16_round`` against an independent implementation of the cast (PyTorch's CPU
  float32 -> bfloat16 conversion) and against hand-computed ties;
* rules R1 (operands) and R2 (the forward result z) on worked examples whose values
  are computed by hand;
* the decomposition of reading c25 on a small RevNet-18 chain: the bf16 arithmetic
  with the exact ReLU masks replayed stays within 2e-2 of the exact oracle on every
  tensor, while its own masks differ from the exact ones in a small counted fraction
  of decisions and account for the rest of the gap on the gradients.
"""
import numpy as np
import pytest

from oracle import primitives as P

torch = pytest.importorskip("torch")


def _torch_bf16(x32):
    return torch.from_numpy(np.ascontiguousarray(x32, np.float32)).to(torch.bfloat16).double().numpy()


def test_bf16_round_matches_torch_cast_over_all_magnitudes():
    g = np.random.default_rng(0)
    with np.errstate(over="ignore"):   # the largest draws overflow fp32 to inf on purpose
        x = (g.standard_normal(200_000) * np.exp2(g.integers(-149, 128, 200_000))).astype(np.float32)
    np.testing.assert_array_equal(P.bf16_round(x), _torch_bf16(x))


def test_bf16_round_special_values():
    f32 = np.finfo(np.float32)
    x = np.array([0.0, -0.0, np.inf, -np.inf, f32.max, -f32.max, f32.tiny, f32.tiny / 3, 1e-45, -1e-45,
                  3.3895314e38, 3.3961775e38, 1.0, -1.0], np.float32)
    got, want = P.bf16_round(x), _torch_bf16(x)
    np.testing.assert_array_equal(got, want)
    assert np.isnan(P.bf16_round(np.array([np.nan], np.float32)))[0]
    assert np.isinf(got[4])          # fp32 max rounds past the largest bf16: overflow to inf


def test_bf16_round_ties_to_even_by_hand():
    # bf16 spacing on [1, 2) is 2^-7: 1 + 2^-8 is a tie between 1 (even) and 1 + 2^-7 (odd)
    assert P.bf16_round(np.float32(1 + 2 ** -8)) == 1.0
    # 1 + 3 * 2^-8 ties between 1 + 2^-7 (odd) and 1 + 2^-6 (even)
    assert P.bf16_round(np.float32(1 + 3 * 2 ** -8)) == 1 + 2 ** -6
    # just above the tie rounds up
    assert P.bf16_round(np.float32(1 + 2 ** -8 + 2 ** -20)) == 1 + 2 ** -7
    # spacing on [2, 4) is 2^-6: 3 + 3 * 2^-7 = 193.5 * 2^-6 -> 194 * 2^-6 = 3.03125
    assert P.bf16_round(np.float32(3 + 3 * 2 ** -7)) == 3.03125


def test_rule_r1_rounds_conv_operands():
    """1x1 conv of one pixel: x = 1 + 2^-8 (rounds to 1), w = 3 -> z = 3 under R1,
    3 + 3 * 2^-8 in exact arithmetic."""
    x = np.full((1, 1, 1, 1), 1 + 2 ** -8)
    w = np.full((1, 1, 1, 1), 3.0)
    assert P.conv2d(x, w)[0, 0, 0, 0] == 3 + 3 * 2 ** -8
    with P.bf16_convolutions():
        assert P.conv2d(x, w)[0, 0, 0, 0] == 3.0
    assert P.conv2d(x, w)[0, 0, 0, 0] == 3 + 3 * 2 ** -8        # the mode is scoped


def test_rule_r2_rounds_the_forward_result():
    """Operands exactly representable in bf16 (1 and 1 + 2^-7), three channels:
    z = 3 + 3 * 2^-7 exactly, which is not a bf16 value; R2 stores it as 3.03125."""
    x = np.ones((1, 3, 1, 1))
    w = np.full((1, 3, 1, 1), 1 + 2 ** -7)
    assert P.conv2d(x, w)[0, 0, 0, 0] == 3 + 3 * 2 ** -7
    with P.bf16_convolutions():
        assert P.conv2d(x, w)[0, 0, 0, 0] == 3.03125


def test_rule_r1_rounds_vjp_operands_but_not_results():
    """dgrad = dout * w and wgrad = dout * x with dout = 1 + 2^-8 (rounds to 1):
    under R1 both see dout = 1; the results themselves are not rounded (R3):
    w = x = 1 + 2^-7 gives 1 + 2^-7 for each."""
    x = np.full((1, 1, 1, 1), 1 + 2 ** -7)
    w = np.full((1, 1, 1, 1), 1 + 2 ** -7)
    dout = np.full((1, 1, 1, 1), 1 + 2 ** -8)
    dx, dw = P.conv2d_vjp(x, w, 1, 0, dout)
    assert dx[0, 0, 0, 0] == (1 + 2 ** -8) * (1 + 2 ** -7)
    with P.bf16_convolutions():
        dx, dw = P.conv2d_vjp(x, w, 1, 0, dout)
    assert dx[0, 0, 0, 0] == 1 + 2 ** -7 and dw[0, 0, 0, 0] == 1 + 2 ** -7


def test_rule_r3_leaves_bn_relu_and_linear_exact():
    z = np.random.default_rng(1).standard_normal((4, 3, 2, 2)) * (1 + 2 ** -9)
    with P.bf16_convolutions():
        a, _ = P.bn_train_forward(z, np.ones(3), np.zeros(3))
        r, _ = P.relu(z)
        y = P.linear(z.reshape(4, -1), np.eye(12) * (1 + 2 ** -9), np.zeros(12))
    b, _ = P.bn_train_forward(z, np.ones(3), np.zeros(3))
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(r, np.maximum(z, 0))
    np.testing.assert_array_equal(y, z.reshape(4, -1) * (1 + 2 ** -9))


def test_mask_replay_reproduces_the_recorded_run():
    """Recording then replaying the masks of the same computation changes nothing."""
    a = np.random.default_rng(2).standard_normal((5, 7))
    P.MASKS["record"] = rec = []
    y1, m1 = P.relu(a)
    P.MASKS["record"] = None
    P.MASKS["replay"] = list(rec)
    y2, m2 = P.relu(a + 1e-3)     # a different input, the recorded decisions
    P.MASKS["replay"] = None
    np.testing.assert_array_equal(m1, m2)
    np.testing.assert_array_equal(y2, np.where(m1, a + 1e-3, 0.0))


def test_c25_decomposition_small_revnet18_chain():
    """Reading c25 on RevNet-18 / 32x32 / batch 4, J = 4 (the bench partition): the
    bf16 rule with the exact masks replayed is within 2e-2 of exact everywhere; with
    its own masks, a counted fraction of decisions flips and the gradients move
    further, while the forward, x~ and theta stay within 2e-2."""
    from tests import fullsize_oracle as FO
    from tests.gpu_harness import rel
    FO.WORKLOADS.setdefault("r18_b4_j4", ("revnet18", 32, 10, 4, [5, 4, 4, 5], 5e-4))
    units0, counts, inputs, recs, flips = FO.chain("r18_b4_j4")
    frac = {k: sum(f for f, _ in v.values()) / sum(n for _, n in v.values()) for k, v in flips.items()}
    assert 1e-5 < frac["bf16_vs_exact"] < 1e-2, flips
    # another summation order of the same arithmetic moves far fewer decisions
    assert frac["exact_acc32_vs_exact"] < frac["bf16_vs_exact"] / 20, frac
    assert frac["bf16_acc32_vs_bf16"] < frac["bf16_vs_exact"] / 5, frac
    for j in range(1, len(counts) + 1):
        ex, bq, pq = recs["exact"][j], recs["bf16"][j], recs["pinned"][j]
        for key in ("fwd", "xt", "d"):
            if ex[key] is None:
                continue
            for h in range(len(ex[key])):
                assert rel(pq[key][h], ex[key][h]) <= 2e-2, (j, key, h)
                if key != "d":
                    assert rel(bq[key][h], ex[key][h]) <= 2e-2, (j, key, h)
        for key in ("grads", "v", "theta", "buffers"):
            for a, b in zip(pq[key], ex[key]):
                assert rel(a, b) <= 2e-2, (j, key)
        for a, b in zip(bq["theta"], ex["theta"]):
            assert rel(a, b) <= 2e-2, (j, "theta")
