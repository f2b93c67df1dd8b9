"""The NCCL transport across GPUs (PETRA_TRANSPORT_NCCL), when the box has >= 2.

torchrun launches tests/nccl_pipeline_worker.py with one rank per GPU (world 2 and,
with >= 4 GPUs, 4); each rank's stages must be bitwise equal to a world-1 pipeline of
the same model and inputs.  On a one-GPU box the same schedule / event / overlap code
is covered by tests/test_multirank_local_gpu.py (PETRA_TRANSPORT_LOCAL)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_transport_bitwise_equal_world_1(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world),
           os.path.join(ROOT, "tests", "nccl_pipeline_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("bitwise equal to world 1: True") == world, r.stdout
