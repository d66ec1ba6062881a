"""Node visits and leaf tests per ray-bounce of the instrumented trace kernel
(RR_TRACE_COUNT) for each traversal tree, plus the uninstrumented kernel time:
python profiles/trace_counts.py c5 [stride]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, _lib  # noqa: E402
from paper_1811_05784_b200 import roomray as rr  # noqa: E402
from paper_1811_05784_b200 import scenes  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    stride = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    s = scenes.CONFIGS[name]()
    ctx = Context(0)
    tree = rr.AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    cfg = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    recv = [Receiver(*r) for r in s.receivers]
    sub = dict(first=0, stride=stride) if stride else {}
    for label, fl in (("tree8", _lib.RR_TRACE_TREE8), ("tree2", _lib.RR_TRACE_TREE2)):
        t = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), recv, cfg, flags=fl, **sub)
        ms = t.kernel_ms
        c = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), recv, cfg, flags=fl | _lib.RR_TRACE_COUNT,
                            **sub).stats
        rb = c.ray_bounces
        print(f"{name} {label}: {rb} rb, kernel {ms:.3f} ms ({rb / ms / 1e6:.3f} G rb/s), "
              f"node visits/rb {c.node_visits / rb:.2f}, leaf tests/rb {c.leaf_tests / rb:.2f}")


if __name__ == "__main__":
    main()
