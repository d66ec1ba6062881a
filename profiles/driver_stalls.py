"""Latency distribution of a small C-ABI call (rr_fibonacci_directions, 1000
rays: allocation, one kernel, copy back, free) repeated for 30 s on the box.
Round 2: 1.18e6 calls, median 0.025 ms, p99 0.030 ms, max 13.9 ms, one call
over 5 ms -- the 30-300 ms stalls seen in the C5 e2e loop do not come from
per-call driver overhead of this kind."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1811_05784_b200 import roomray as rr, Context
ctx = Context(0)
lat = []
t_end = time.time() + 30
while time.time() < t_end:
    t = time.perf_counter()
    rr.fibonacci_directions(1000, ctx=ctx)
    lat.append(time.perf_counter() - t)
lat = np.array(lat) * 1e3
print(f"calls {len(lat)} median {np.median(lat):.3f} ms p99 {np.percentile(lat, 99):.3f} max {lat.max():.1f} ms; >5 ms: {(lat > 5).sum()}, >50 ms: {(lat > 50).sum()}")
