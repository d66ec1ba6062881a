"""The checked build under the traversal, the tree builders, K5 and the
exchange pipeline.  compute-sanitizer is closed on this GPU pool (runs under
it left GPUs needing a reset), so memory safety is checked by the library's
own device-side bounds checks instead: libroomray_b200_checked.so is the
same sources with -DRR_CHECKED, where RR_DCHECK guards the traversal stack
depths (binary, 4-wide, 8-wide), node and face indices, the face-history
writes and the 8-wide builder's face copies, and traps on a violation.  The
workload (tests/native/checked_run.py) also compares C1 with the oracle on
every traversal tree, so the checks run on the exact path."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1811_05784_b200", "libroomray_b200_checked.so")


def test_checked_build_runs_clean():
    assert os.path.exists(CHECKED), "build the checked library (make -C paper_1811_05784_b200/csrc)"
    env = dict(os.environ, RR_LIB_PATH=CHECKED)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "native", "checked_run.py")], capture_output=True,
                       text=True, timeout=900, env=env)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "RR_DCHECK failed" not in out, out[-4000:]
    assert "checked workload ok" in p.stdout, out[-4000:]
