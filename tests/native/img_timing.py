import sys, time; sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes
s = scenes.config2()
tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption))
for i in range(2):
    dt = rr.trace_device(tree, rr.SourceConfig(s.source, s.ray_count), rr.Receiver(*s.receivers[0]), rr.TraceConfig(max_iterations=50, max_range=686.0))
    t = time.time(); im = rr.build_image_sources_device(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True)); print("images", im.n, time.time() - t, "captures", dt.stats.n_captures, file=sys.stderr)
