import os, sys
sys.path.insert(0, os.getcwd())
from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, scenes
from paper_1811_05784_b200 import roomray as rr
s = scenes.config5()
ctx = Context(0)
tree = rr.AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
dt = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), [Receiver(*r) for r in s.receivers],
                     TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range))
for i in range(int(sys.argv[1])):
    im = rr.build_image_sources_device(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True))
    del im
