"""Time per bounce vs number of bounces (does warp coherence decay?)."""
import sys; sys.path.insert(0,'.')
from paper_1811_05784_b200 import roomray as rr, scenes
s=scenes.config2()
tree=rr.AccelTree(rr.TriangleMesh(s.vertices,s.faces,s.absorption))
import os
for order in ("1","0"):
    os.environ["RR_ORDER"]=order
    for it in (1,2,5,10,20,50):
        best=1e9
        for k in range(3):
            dt=rr.trace_device(tree, rr.SourceConfig(s.source, s.ray_count), rr.Receiver(*s.receivers[0]), rr.TraceConfig(max_iterations=it, max_range=s.max_range))
            best=min(best, dt.kernel_ms)
        print(f"order={order} iters={it:3d} kernel {best:8.3f} ms  {dt.stats.ray_bounces/best/1e6:6.3f} G rb/s", flush=True)
