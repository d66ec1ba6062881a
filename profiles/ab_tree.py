"""Tree-builder A/B: for each environment setting (the builder's runtime
switches, e.g. RR_SAH_FIN=1,RR_SAH_MIN=17), in its own process: scene build
time, node visits and leaf tests per ray-bounce of the 8-wide traversal on a
lattice subset (RR_TRACE_COUNT), and the full-lattice trace kernel time.
    python profiles/ab_tree.py c5 "" RR_SAH_FIN=1 RR_SAH_MIN=17,RR_SAH_FIN=1"""
import os
import subprocess
import sys

CHILD = r"""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, _lib, scenes
from paper_1811_05784_b200 import roomray as rr
s = scenes.CONFIGS[sys.argv[1]]()
ctx = Context(0)
mesh = TriangleMesh(s.vertices, s.faces, s.absorption)
bt = []
for _ in range(3):
    t0 = time.perf_counter(); tree = rr.AccelTree(mesh, ctx); ctx.synchronize() if hasattr(ctx, 'synchronize') else None
    bt.append((time.perf_counter() - t0) * 1e3)
cfg = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
recv = [Receiver(*r) for r in s.receivers]
c = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), recv, cfg, flags=_lib.RR_TRACE_COUNT, first=0, stride=8).stats
ms = [rr.trace_device(tree, SourceConfig(s.source, s.ray_count), recv, cfg).kernel_ms for _ in range(3)]
rb = c.ray_bounces
print(f"[{os.environ.get('RR_AB_TAG', '')}] build {min(bt):.1f} ms; visits/rb {c.node_visits / rb:.3f} leaf tests/rb {c.leaf_tests / rb:.3f} "
      f"(stride 8, {rb} rb); kernel min {min(ms):.2f} ms {sorted(ms)}")
"""

for extra in sys.argv[2:]:
    env = dict(os.environ, RR_AB_TAG=extra)
    env.update(kv.split("=", 1) for kv in extra.split(",") if kv)
    subprocess.run([sys.executable, "-c", CHILD, sys.argv[1]], env=env, check=False)
