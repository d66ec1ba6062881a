"""A/B timing of traversal variants on one config (development tool).

    python tests/native/ab_trace.py c2 binary,f32,wide      (RR_MINB=6/8/10 env)
"""
import os
import sys

sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes, _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["binary", "f32", "wide"]
s = scenes.CONFIGS[cfg]()
tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
flags = {"binary": 0, "f32": _lib.RR_TRACE_F32_LEAVES, "wide": _lib.RR_TRACE_WIDE | _lib.RR_TRACE_NO_SMEM_CACHE,
         "wide+smem": _lib.RR_TRACE_WIDE}
for name in variants:
    ms = []
    for i in range(4):
        dt = rr.trace_device(tree, rr.SourceConfig(s.source, s.ray_count), rr.Receiver(*s.receivers[0]),
                             rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                             flags=flags[name])
        ms.append(dt.kernel_ms)
        nc = dt.stats.n_captures
    best = min(ms[1:])
    print(f"{cfg} {name:10s} MINB={os.environ.get('RR_MINB', '8'):3s} kernel {best:8.3f} ms  "
          f"{dt.stats.ray_bounces / best / 1e6:6.3f} G ray-bounces/s  captures {nc}", flush=True)
