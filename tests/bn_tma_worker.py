"""Subprocess of tests/test_bn_tma_gpu.py: one stage tick (forward, backward + update)
of a named case, outputs saved to an .npz.  The BN kernels the library picks depend on
PETRA_BN_TMA_{APPLY,REDUCE,DZ} (read once per process), so each setting runs here."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle.units import Branch, ConvBN, DSUnit, RevUnit, StemUnit  # noqa: E402
from paper_2406_02052_b200 import Stage, _lib as L, models as PM  # noqa: E402
from tests.gpu_harness import nhwc, oracle_to_product_units, pack_params, rand_params  # noqa: E402


def rev(c, dst):
    return RevUnit(dst, Branch([ConvBN(c, c, 3, 1)]))


CASES = {
    # stem: split dy halves (cs > 0) in the BN backward; M = 3 * 10 * 10 = 300 rows (ragged chunks)
    "stem_rev_ragged": (lambda: [StemUnit(3, 128, 3, 1, False), rev(64, 0), rev(64, 1)], 3, (10, 10, 3), L.BF16_TC),
    # many row blocks per channel tile (nrb > 1), bf16 z, coupling addend
    "rev_pair_b64": (lambda: [rev(64, 0), rev(64, 1)], 64, (32, 32, 64), L.BF16_TC),
    # fp32 z (SIMT convolutions)
    "rev_pair_fp32_ragged": (lambda: [rev(64, 0), rev(64, 1)], 3, (10, 10, 64), L.FP32),
    # DS unit: projections without ReLU, strided operand views
    "ds_rev": (lambda: [DSUnit(0, Branch([ConvBN(64, 128, 3, 2)]), ConvBN(64, 128, 1, 2, relu=False),
                               ConvBN(64, 128, 1, 2, relu=False)), rev(128, 1)], 6, (14, 14, 64), L.BF16_TC),
    # ImageNet-style stem: 7x7 / 2 conv + BN-ReLU + 3x3 / 2 max-pool, then a reversible unit
    "stem_maxpool": (lambda: [StemUnit(3, 128, 7, 2, True), rev(64, 0)], 2, (32, 32, 3), L.BF16_TC),
}


def main(case, out):
    make, B, hwc, prec = CASES[case]
    units = rand_params(make(), 3)
    torch.cuda.set_device(0)
    st = Stage(PM.StageSpec(oracle_to_product_units(units), B, hwc, prec, fifo_capacity=3), seed=0)
    th, bf = pack_params(units)
    st.set_params(th, np.zeros_like(th), bf)
    stem = hwc[2] == 3
    H, W, C = hwc
    xs = [torch.tensor(nhwc(synth.images((B, C, H, W), 0, h)), dtype=torch.float32, device="cuda")
          for h in range(1 if stem else 2)]
    o = [torch.empty(st.out_shape, device="cuda") for _ in range(2)]
    st.forward(0, xs[0], None if stem else xs[1], o[0], o[1])
    d = [torch.tensor(synth.normal(tuple(st.out_shape), 8, h), dtype=torch.float32, device="cuda") for h in range(2)]
    res = [torch.empty((B, H, W, C), device="cuda") for _ in range(4)]
    if stem:
        st.backward(0, o[0], o[1], d[0], d[1], None, None, None, None, 0.05)
    else:
        st.backward(0, o[0], o[1], d[0], d[1], *res, 0.05)
    torch.cuda.synchronize()
    th, v, bfs = st.get_params()
    arrs = {"o0": o[0].cpu().numpy(), "o1": o[1].cpu().numpy(), "theta": th, "v": v, "running": bfs,
            "grads": st.get_grads()}
    if not stem:
        for k in range(4):
            arrs[f"r{k}"] = res[k].cpu().numpy()
    # the evaluation forward (BN on the running statistics) of the same stage
    oe = [torch.empty(st.out_shape, device="cuda") for _ in range(2)]
    st.eval(xs[0], None if stem else xs[1], oe[0], oe[1])
    torch.cuda.synchronize()
    arrs["eval0"], arrs["eval1"] = oe[0].cpu().numpy(), oe[1].cpu().numpy()
    np.savez(out, **arrs)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
