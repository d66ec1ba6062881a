"""Workload for tests/test_gpu_sanitizer.py (run under compute-sanitizer):
C1 trace on every traversal tree (binary, 4-wide, 8-wide), a 20 000-ray
subset of C3 (scene build incl. SAH + wide collapses), image sources with
coplanar merge, the IR stage and the one-rank exchange pipeline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_1811_05784_b200 import (AccelTree, Context, Receiver, SourceConfig, TraceConfig,  # noqa: E402
                                   TriangleMesh, _lib, scenes)
from paper_1811_05784_b200 import roomray as rr  # noqa: E402


def main():
    ctx = Context(0)
    s = scenes.config1()
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    cfg = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    for fl in (0, _lib.RR_TRACE_TREE8, _lib.RR_TRACE_TREE2):
        dt = rr.trace_device(tree, SourceConfig(s.source, 4000), [Receiver(*s.receivers[0])], cfg, flags=fl)
        im = rr.build_image_sources(dt, 4000, rr.AirModel(), rr.ClusterOptions(1e-6, True))
        assert len(im.distance) > 0
    comm = rr.Comm(ctx, rr.Comm.unique_id(), 1, 0)
    res = rr.pipeline_sharded(tree, SourceConfig(s.source, 4000), [Receiver(*s.receivers[0])], cfg, comm=comm,
                              sample_rate=s.sample_rate, length=int(s.sample_rate))
    assert res.ray_bounces > 0
    c3 = scenes.config3()
    t3 = AccelTree(TriangleMesh(c3.vertices, c3.faces, c3.absorption), ctx)
    c3cfg = TraceConfig(max_iterations=c3.max_iterations, max_range=c3.max_range)
    recs = [Receiver(*r) for r in c3.receivers]
    for fl in (0, _lib.RR_TRACE_TREE8):
        dt = rr.trace_device(t3, SourceConfig(c3.source, c3.ray_count), recs, c3cfg, first=0, stride=50, flags=fl)
        rr.build_image_sources(dt, c3.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True), receiver=0)
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
