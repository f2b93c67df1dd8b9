"""compute-sanitizer over the mbarrier / TMA / tcgen05 kernels (SURVEY 4.2 tier T5;
VERDICT r1 "next round" 7): memcheck (out-of-bounds / misaligned accesses), racecheck
(shared-memory hazards) and synccheck (barrier misuse) on tests/sanitizer_target.py,
each required to report 0 errors.

Opt-in (PETRA_SANITIZER=1): the GPU pool this repository is measured on has closed
compute-sanitizer (runs under it left GPUs needing a reset), so by default the tier is
skipped; where the tool is usable the test runs it and requires a clean report."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.skipif(os.environ.get("PETRA_SANITIZER", "0") != "1",
                    reason="compute-sanitizer is closed on the measurement pool; set PETRA_SANITIZER=1 to run")
def test_compute_sanitizer_clean(tool):
    env = dict(os.environ, PETRA_GRAPHS="0")  # plain launches: every kernel attributed by name
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20", "--target-processes", "all",
           sys.executable, os.path.join(ROOT, "tests", "sanitizer_target.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out", "sanitizer"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "sanitizer", f"{tool}.log"), "w") as f:
        f.write(out)
    if "sanitizer target done" not in out and "closed" in out:
        pytest.skip(out.strip()[:300])
    assert "sanitizer target done" in out, out[-4000:]
    clean = ("ERROR SUMMARY: 0 errors" in out) or ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out)
    assert r.returncode == 0 and clean, out[-6000:]
