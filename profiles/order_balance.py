"""Per-rank image-stage load of the order-class ownership (shard.py /
rr_shard.cu assign_orders) for a config at world sizes 2..8: captures per
order class of each receiver from one device trace, LPT assignment, and the
largest rank's share against a perfect split.  python profiles/order_balance.py c3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, scenes  # noqa: E402
from paper_1811_05784_b200 import roomray as rr  # noqa: E402
from paper_1811_05784_b200.shard import assign_orders  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    s = scenes.CONFIGS[name]()
    ctx = Context(0)
    tree = rr.AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    c = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), [Receiver(*r) for r in s.receivers],
                        TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)).captures()
    order = np.diff(c.hist_off)
    units = []  # (count, receiver, order) over all receivers: the joint ownership of rr_shard.cu
    for r in range(len(s.receivers)):
        cnt = np.bincount(order[c.recv == r], minlength=s.max_iterations + 1)
        units += [(int(cnt[o]), r, o) for o in range(len(cnt))]
    line = []
    for world in (2, 4, 8):
        load = np.zeros(world)
        for n, r, o in sorted(units, key=lambda u: (-u[0], u[1], u[2])):
            q = int(np.argmin(load))
            load[q] += n
        line.append(f"w{world}: max/mean {load.max() / max(load.mean(), 1):.2f}")
    print(f"{name} all {len(s.receivers)} receivers jointly ((receiver, order) units): " + ", ".join(line))
    for r in range(len(s.receivers)):
        counts = np.bincount(order[c.recv == r], minlength=s.max_iterations + 1)
        line = []
        for world in (2, 4, 8):
            own = assign_orders([int(x) for x in counts], world)
            load = np.zeros(world)
            for o, q in enumerate(own):
                load[q] += counts[o]
            line.append(f"w{world}: max/mean {load.max() / max(load.mean(), 1):.2f}")
        top = np.argsort(-counts)[:4]
        print(f"{name} receiver {r}: {counts.sum()} captures, top orders {list(top)} "
              f"({[int(counts[t]) for t in top]}); " + ", ".join(line))


if __name__ == "__main__":
    main()
