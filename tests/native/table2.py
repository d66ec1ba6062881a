"""The paper's complexity benchmark (Table 2; the reference's
`roomray bench`, bench.cpp:71-102) on the GPU: N = M = 2^k rays and faces,
rays from the centre of a subdivided tetrahedron, receiver far outside,
unbounded range; per-iteration device time of step() with the SAH tree and
with brute force (nearest_hit_brute), after one warm-up iteration.

    python tests/native/table2.py [k_min k_max brute_max]   (default 10 20 16)

Beside it, the reference's own step() (oracle/_ref, bench.cpp's timing loop)
on this host's cores: tree rows up to k_max, brute force up to k = 14.
"""
import math
import os
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_05784_b200 import roomray as rr, scenes  # noqa: E402
import oracle  # noqa: E402  (reference CPU column only)

PAPER = {10: (0.20, 0.26), 11: (0.21, 0.44), 12: (0.25, 0.91), 13: (0.30, 3.05), 14: (0.33, 11.44),
         15: (0.48, 45.3), 16: (0.77, 181.61), 17: (1.85, 725.17), 18: (2.76, 2927.9), 19: (8.36, None),
         20: (13.78, None)}


def per_iteration(tree, n, brute, repeats):
    src = rr.SourceConfig((0.0, 0.0, 0.0), n)
    host = rr.Rays.emit(src, hist_cap=repeats + 2)
    rays = rr.Rays(*[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in
                     (host.origin, host.dir, host.mult, host.path, host.alive, host.hist, host.n_hist)])
    recv = rr.Receiver((1e6, 1e6, 1e6), 1e-3)
    cfg = rr.TraceConfig(max_range=1e30)
    rr.step(tree, rays, recv, cfg, brute=brute)  # warm-up
    ms = [rr.step(tree, rays, recv, cfg, brute=brute).kernel_ms for _ in range(repeats)]
    return float(np.mean(ms)) / 1e3


def main():
    kmin, kmax, bmax = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10, 20, 16)))
    ref = oracle.Ref() if oracle.ref_available() else None
    threads = os.cpu_count() or 1
    rows = []
    f3 = lambda x: '%.3e' % x if x else '—'  # noqa: E731
    print(f"reference CPU column: oracle/_ref step() with thread_count={threads}" if ref else "reference not built")
    print("| k | faces = rays | depth | B200 build (s) | B200 step, tree (s) | B200 step, brute (s) | "
          "ref build (s) | ref step, tree (s) | ref step, brute (s) | paper tree (s) | paper brute (s) | "
          "B200 vs ref, tree |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for k in range(kmin, kmax + 1):
        v, f, a = scenes.subdivided_tetrahedron(k)
        mesh = rr.TriangleMesh(v, f, a)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tree = rr.AccelTree(mesh)
        torch.cuda.synchronize()
        b_build = time.perf_counter() - t0
        t_tree = per_iteration(tree, 1 << k, False, 10)
        t_brute = per_iteration(tree, 1 << k, True, 2) if k <= bmax else None
        r_tree = r_brute = r_build = None
        if ref:
            r_tree, r_build, _ = ref.bench_row(k, True, threads, 0.25, 50)
            if k <= 14:
                r_brute = ref.bench_row(k, False, threads, 0.25, 5)[0]
        rows.append((k, t_tree, t_brute))
        pt, pb = PAPER.get(k, (None, None))
        print(f"| {k} | {1 << k} | {tree.depth()} | {b_build:.3e} | {t_tree:.3e} | {f3(t_brute)} | {f3(r_build)} | "
              f"{f3(r_tree)} | {f3(r_brute)} | {pt if pt else '—'} | {pb if pb else '—'} | "
              f"{'%.0f' % (r_tree / t_tree) if r_tree else '—'} |", flush=True)

    def slope(pts):
        x = np.array([math.log2(1 << k) for k, _ in pts])
        y = np.array([math.log2(t) for _, t in pts])
        return np.polyfit(x, y, 1)[0]

    print(f"\nlog-log slope of time vs N=M: tree {slope([(k, t) for k, t, _ in rows]):.2f}, "
          f"brute {slope([(k, b) for k, _, b in rows if b]):.2f} (paper: tree 0.60 over k=12..18, "
          f"brute 1.38 over k=10..14)")


if __name__ == "__main__":
    main()
