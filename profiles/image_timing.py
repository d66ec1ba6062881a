"""C5 image-source stage alone: wall time of build_image_sources_device
(device-resident captures in, device image lists out), first call after a
fresh trace vs repeats on the same trace.  RR_TIMING=1 adds the library's
per-stage event times (and host-side statistics, which slow it)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, scenes
from paper_1811_05784_b200 import roomray as rr
torch.cuda.synchronize()
s = scenes.config5()
ctx = Context(0)
tree = rr.AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t = time.perf_counter()
    dt = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), [Receiver(*r) for r in s.receivers],
                         TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range))
    torch.cuda.synchronize()
    print(f"trace {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
    for i in range(2):
        t = time.perf_counter()
        im = rr.build_image_sources_device(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True))
        torch.cuda.synchronize()
        print(f"  images {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
        del im
    del dt
