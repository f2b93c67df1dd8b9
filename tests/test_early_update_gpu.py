"""Early per-unit updates (PETRA_EARLY_UPDATE=1, the default) move each unit's
Nesterov update onto the wgrad stream right after the unit's backward instead of one launch at
the end of the stage's tick.  Same kernel, same per-element arithmetic, so a RevNet-18 J=4
pipeline must give BITWISE the same losses, theta, v and running statistics either way (fp32 and
bf16 paths); each setting runs in its own process."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(prec, early, path):
    env = dict(os.environ, PETRA_EARLY_UPDATE="1" if early else "0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "early_update_worker.py"), prec, path], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return dict(np.load(path))


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_early_updates_bitwise_equal_end_of_tick_update(prec, tmp_path):
    a = _run(prec, True, str(tmp_path / "early.npz"))
    b = _run(prec, False, str(tmp_path / "late.npz"))
    assert sorted(a) == sorted(b) and len(a) > 6
    for k in a:
        assert np.array_equal(np.atleast_1d(a[k]).view(np.uint8), np.atleast_1d(b[k]).view(np.uint8)), k
