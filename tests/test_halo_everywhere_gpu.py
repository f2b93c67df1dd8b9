"""The halo convolution (and halo wgrad) on EVERY 3x3 stride-1 layer, whatever its
grid size or zero-border overhead (PETRA_HALO_MIN_WORK=1, PETRA_HALO_MAX_PAD=1000):
the stage parity suite and the full-size tail test run in a subprocess with those
knobs (they are read once per process).  This covers the halo paths the default
plan never selects for the benchmark models -- N tiles narrower than N (BN = 256
for 512 output channels: one BN-partial row slice per CTA), 4x4 / 7x7 grids whose
border more than doubles the rows -- against the same oracle bars as the default
path."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_stage_parity_with_halo_on_every_3x3_layer():
    env = dict(os.environ, PETRA_HALO_MIN_WORK="1", PETRA_HALO_MAX_PAD="1000")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           "tests/test_parity_gpu.py", "tests/test_fullsize_gpu.py", "tests/test_kernels_gpu.py", "-k",
           "stage or tail or padded"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
