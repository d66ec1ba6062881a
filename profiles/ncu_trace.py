"""One trace of a BASELINE config on cuda:0, for ncu captures of the trace
kernel (profiles/ncu_trace_<config>.csv, read by bench.py's roofline):

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum \
      -k regex:trace_kernel --clock-control none --csv --page raw --print-units base \
      python profiles/ncu_trace.py c5 > profiles/ncu_trace_c5.csv
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh  # noqa: E402
from paper_1811_05784_b200 import roomray as rr  # noqa: E402
from paper_1811_05784_b200 import scenes  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    stride = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # lattice subset k = 0 mod stride
    s = scenes.CONFIGS[name]()
    ctx = Context(0)
    tree = rr.AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    cfg = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    for _ in range(reps):
        dt = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), [Receiver(*r) for r in s.receivers], cfg,
                             **(dict(first=0, stride=stride) if stride else {}))
        print(f"{name}: {dt.stats.ray_bounces} ray*bounces, kernel {dt.kernel_ms:.3f} ms", file=sys.stderr)
        del dt


if __name__ == "__main__":
    main()
