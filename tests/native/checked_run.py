"""Workload for tests/test_gpu_checked.py, run against the checked build
(RR_LIB_PATH=libroomray_b200_checked.so: device-side bounds checks on stack
depths and node / face / history indices, which trap on failure): C1 traced
on every traversal tree (binary, 8-wide; C3 below also the 4-wide) and
compared with the oracle capture for capture, image sources with coplanar
merge, the one-rank NCCL exchange pipeline, a 20 000-ray subset of C3 with
its scene build (SAH tree, 4-wide and 8-wide collapses)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_1811_05784_b200 import (AccelTree, Context, Receiver, SourceConfig, TraceConfig,  # noqa: E402
                                   TriangleMesh, _lib, scenes)
from paper_1811_05784_b200 import roomray as rr  # noqa: E402
import numpy as np  # noqa: E402
import oracle  # noqa: E402


def main():
    ctx = Context(0)
    s = scenes.config1()
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    cfg = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    assert os.environ.get("RR_LIB_PATH", "").endswith("_checked.so"), "run against the checked build"
    oc, _ = oracle.Port().scene(oracle.Mesh(s.vertices, s.faces, s.absorption)).trace(
        s.source, 4000, [s.receivers[0][0]], [s.receivers[0][1]], s.max_iterations, s.max_range)
    for fl in (0, _lib.RR_TRACE_TREE8, _lib.RR_TRACE_TREE2):
        dt = rr.trace_device(tree, SourceConfig(s.source, 4000), [Receiver(*s.receivers[0])], cfg, flags=fl)
        g = dt.captures()
        assert len(g) == len(oc) > 0
        for k in ("ray", "path", "point", "mult", "hist"):
            assert np.array_equal(getattr(g, k), getattr(oc, k)), (fl, k)
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
    for fl in (0, _lib.RR_TRACE_TREE8, _lib.RR_TRACE_TREE2):
        dt = rr.trace_device(t3, SourceConfig(c3.source, c3.ray_count), recs, c3cfg, first=0, stride=50, flags=fl)
        rr.build_image_sources(dt, c3.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True), receiver=0)
    print("checked workload ok")


if __name__ == "__main__":
    main()
