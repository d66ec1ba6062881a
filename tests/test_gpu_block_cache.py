"""The context-stream block cache (rr_internal.cuh DevBuf, rr_api.cu) does
not change results.

Every other GPU test runs with the cache on (the default).  Here the C2
pipeline (trace -> image sources with coplanar merge -> 8-band IRs) runs three
times in one process -- the second and third reuse the first run's blocks --
and in subprocesses with the cache off (RR_BLOCK_CACHE_MB=0) and with a 1 MB
cap (every release past the cap evicts the oldest block); all digests must be
equal.  The cache setting is read once per process, hence the subprocesses.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1811_05784_b200 import AccelTree, Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, scenes
from paper_1811_05784_b200 import roomray as rr
s = scenes.CONFIGS["c2"]()
ctx = Context(0)
tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
L = int(round(0.5 * s.sample_rate))
out = []
for rep in range(int(sys.argv[2])):
    res = rr.pipeline_sharded(tree, SourceConfig(s.source, 200000), [Receiver(*r) for r in s.receivers],
                              TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                              options=rr.ClusterOptions(1e-6, True), sample_rate=s.sample_rate, length=L, taps=511)
    h = hashlib.sha256(str(res.ray_bounces).encode())
    for im in res.images:
        for k in sorted(vars(im)):
            v = getattr(im, k)
            if isinstance(v, np.ndarray):
                h.update(k.encode())
                h.update(np.ascontiguousarray(v).tobytes())
    for b in res.band_ir:
        h.update(np.ascontiguousarray(b).tobytes())
    out.append(h.hexdigest())
print(" ".join(out))
"""


def _run(env_extra, reps):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(reps)], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return out.stdout.split()


def test_block_cache_results_unchanged():
    cached = _run({}, 3)
    assert len(set(cached)) == 1, "repeated pipelines on reused blocks differ"
    assert _run({"RR_BLOCK_CACHE_MB": "0"}, 1) == cached[:1]
    assert _run({"RR_BLOCK_CACHE_MB": "1"}, 2) == cached[:2]
