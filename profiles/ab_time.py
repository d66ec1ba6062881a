"""Trace-kernel A/B timing: each library (RR_LIB_PATH) in its own process,
the full lattice of a config traced `reps` times; prints min / median kernel
ms and the ray*bounces (equal across variants when parity holds).
    python profiles/ab_time.py c5 <lib.so> [<lib.so> ...]   (RR_AB_REPS, default 4)
an argument KEY=VAL[,KEY=VAL...]@<lib.so> also sets environment variables
(the library's runtime A/B switches, e.g. RR_W8V=2@paper_1811_05784_b200/libroomray_b200.so)."""
import os
import subprocess
import sys

CHILD = r"""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, scenes
from paper_1811_05784_b200 import roomray as rr
s = scenes.CONFIGS[sys.argv[1]]()
ctx = Context(0)
tree = rr.AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
cfg = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
recv = [Receiver(*r) for r in s.receivers]
ms, rb, nc = [], set(), set()
for _ in range(int(os.environ.get("RR_AB_REPS", "4"))):
    t = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), recv, cfg)
    ms.append(t.kernel_ms); rb.add(t.stats.ray_bounces); nc.add(t.stats.n_captures)
print(f"{os.environ.get('RR_AB_TAG', '')} {os.environ['RR_LIB_PATH']}: min {min(ms):.2f} med {statistics.median(ms):.2f} ms  rb {sorted(rb)} caps {sorted(nc)}")
"""

for arg in sys.argv[2:]:
    extra, lib = arg.split("@", 1) if "@" in arg else ("", arg)
    env = dict(os.environ, RR_LIB_PATH=os.path.abspath(lib), RR_AB_TAG=extra)
    env.update(kv.split("=", 1) for kv in extra.split(",") if kv)
    subprocess.run([sys.executable, "-c", CHILD, sys.argv[1]], env=env, check=False)
