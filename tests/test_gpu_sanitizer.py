"""compute-sanitizer over the tracer, the tree builders and K5 (SURVEY.md
section 5; the reference runs none).  memcheck (out-of-bounds / misaligned
accesses, leaks of device allocations), racecheck (shared-memory hazards),
synccheck (illegal warp / block synchronisation, e.g. a ballot whose mask
names lanes that do not arrive) on tests/native/sanitize_run.py: C1 on
every traversal tree, a 20 000-ray C3 subset incl. its scene build, image
sources with coplanar merge, the one-rank NCCL exchange pipeline."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.path.join(ROOT, "tests", "native", "sanitize_run.py")


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    cs = _sanitizer()
    cmd = [cs, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    p = subprocess.run(cmd + [sys.executable, RUN], capture_output=True, text=True, timeout=1800)
    tail = (p.stdout + p.stderr)[-4000:]
    assert p.returncode == 0, tail
    assert "sanitize workload ok" in p.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in p.stdout + p.stderr, tail
