"""Trace once, then build C2's image sources twice (development tool, run under
an ncu launch list to see the image stage per kernel)."""
import sys
sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes  # noqa: E402

s = scenes.config2()
tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
dt = rr.trace_device(tree, rr.SourceConfig(s.source, s.ray_count), rr.Receiver(*s.receivers[0]),
                     rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range))
for i in range(2):
    im = rr.build_image_sources_device(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True))
    print("images", im.n, file=sys.stderr)
