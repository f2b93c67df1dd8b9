"""The tensor-core convolution's alternative launch plans, each off by default because it
measured slower in the benchmark step, held to the same parity as the default:
  * cluster split-K (PETRA_CONV_CS=1): the K range of a few-tile layer's tile over the CTAs of
    one thread-block cluster, the fp32 partials pushed to their row owners through distributed
    shared memory and summed in rank order in the same kernel;
  * CTA pairs (PETRA_CONV_PAIR=1, with / without two channel blocks per stage): M = 256 tiles
    on cta_group::2 UMMAs, each CTA of a cluster of 2 loading its 128 A rows and half of B.
A mode is read once per process, so the tensor-core-vs-SIMT parity tests (rel 1e-5 on
bf16-exact inputs; the benchmark's R18 layer 3-4 and R50 layer 4 geometries at b64
included), the plan check and the fused BN statistics tests (rel 1e-6 vs fp64 statistics of
the stored z, masked padding rows included) rerun in a subprocess with it on."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = {
    # at the J >= 4 grid cap (the plan's cost model compares against the capped grid)
    "cluster_split_k": {"PETRA_CONV_CS": "1", "PETRA_CONV_CTAS": "40"},
    "cta_pair_kg2": {"PETRA_CONV_PAIR": "1"},
    "cta_pair_kg1": {"PETRA_CONV_PAIR": "1", "PETRA_CONV_PAIR_KG": "1"},
}


@pytest.mark.parametrize("mode", sorted(MODES))
def test_conv_mode_parity(mode):
    env = dict(os.environ, **MODES[mode])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           "tests/test_kernels_gpu.py::test_tc_conv_vs_simt", "tests/test_kernels_gpu.py::test_conv_mode_plan",
           "tests/test_bn_stats_gpu.py"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "skipped" not in r.stdout.splitlines()[-1], r.stdout[-2000:]
