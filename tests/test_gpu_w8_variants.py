"""The 8-wide tracer's two traversals give the same closest hits.

The default is the group traversal (one stack entry per node, remaining
children in octant order); the sorted-push traversal is the fallback for
trees deeper than the group stack, selectable with RR_W8V=1 (RR_W8V=2: the
group traversal without the nearest-first choice).  The environment switch is
read once per process, so each variant runs in a subprocess and reports a
digest of its captures; they must equal the default's bit for bit (the
default itself is pinned to the oracle in test_gpu_default_path.py and
test_gpu_wide.py).
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh, _lib, scenes, trace

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("ray", "recv", "hist_off", "path", "point", "dir", "mult", "hist")

CHILD = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1811_05784_b200 import AccelTree, Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, _lib, scenes, trace
cfg, stride = sys.argv[2], int(sys.argv[3])
s = scenes.CONFIGS[cfg]()
tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), Context(0))
res = trace(tree, SourceConfig(s.source, s.ray_count), [Receiver(c, r) for c, r in s.receivers],
            TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range), first=1, stride=stride,
            flags=_lib.RR_TRACE_TREE8)
h = hashlib.sha256(str(res.ray_bounces).encode())
for k in %r:
    h.update(np.ascontiguousarray(getattr(res.captures, k)).tobytes())
print(h.hexdigest(), len(res.captures))
""" % (FIELDS,)


def _digest(res):
    h = hashlib.sha256(str(res.ray_bounces).encode())
    for k in FIELDS:
        h.update(np.ascontiguousarray(getattr(res.captures, k)).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("cfg,stride", [("c3", 50), ("c5", 2000)])
@pytest.mark.parametrize("variant", ["1", "2"])
def test_traversal_variants_agree(ctx, cfg, stride, variant):
    s = scenes.CONFIGS[cfg]()
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    res = trace(tree, SourceConfig(s.source, s.ray_count), [Receiver(c, r) for c, r in s.receivers],
                TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range), first=1, stride=stride,
                flags=_lib.RR_TRACE_TREE8)
    assert len(res.captures) > 0
    env = dict(os.environ, RR_W8V=variant)
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, cfg, str(stride)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    digest, n = out.stdout.split()
    assert int(n) == len(res.captures)
    assert digest == _digest(res)
