"""Profiling driver: one warm-up and one timed C2 trace (for ncu captures)."""
import sys

sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = scenes.CONFIGS[cfg]()
tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
for i in range(2):
    dt = rr.trace_device(tree, rr.SourceConfig(s.source, s.ray_count), rr.Receiver(*s.receivers[0]),
                         rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range))
    print(f"trace {i}: {dt.kernel_ms:.3f} ms, {dt.stats.ray_bounces} ray-bounces, "
          f"{dt.stats.ray_bounces / dt.kernel_ms / 1e6:.3f} G/s")
