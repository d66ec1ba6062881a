"""Scene-build stage timings (development tool): RR_TIMING=1 python tests/native/build_timing.py c2"""
import sys
import time

sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes  # noqa: E402

s = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
for i in range(3):
    t = time.perf_counter()
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
    print(f"build {i}: {1e3 * (time.perf_counter() - t):.2f} ms wall, {tree.build_ms:.2f} ms device events",
          file=sys.stderr)
