"""Cluster split-K (PETRA_CONV_CS=1, off by default): the K range of a few-tile
layer's tile over the CTAs of one thread-block cluster, the fp32 partials pushed to their row
owners through distributed shared memory and summed in rank order in the same kernel.  The
mode is read once per process, so the tensor-core-vs-SIMT parity tests (the benchmark's R18
layer 3-4 and R50 layer 4 geometries at b64 included), the plan check and the fused BN
statistics tests (rel 1e-6 vs fp64 statistics of the stored z) rerun in a subprocess with it on."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cluster_split_k_parity():
    env = dict(os.environ, PETRA_CONV_CS="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           "tests/test_kernels_gpu.py::test_tc_conv_vs_simt", "tests/test_kernels_gpu.py::test_cluster_split_plan",
           "tests/test_bn_stats_gpu.py"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "skipped" not in r.stdout.splitlines()[-1], r.stdout[-2000:]
