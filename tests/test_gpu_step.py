"""step() (tracer.hpp:43-45) on the GPU: repeated single iterations over a
caller-held Ray span reproduce trace() of the oracle capture for capture
(bit for bit with the oracle's lattice directions), the brute-force path
(step with tree = nullptr) equals the tree path, and device-resident spans
are updated in place."""
import numpy as np
import pytest
import torch

import oracle
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu


def _concat(parts):
    keys, rows = [], []
    for c in parts:
        for i in range(len(c)):
            rows.append((int(c.ray[i]), float(c.path[i]), c.point[i], c.dir[i], c.mult[i], c.history(i)))
    rows.sort(key=lambda r: (r[0], r[1]))
    return rows


def test_steps_reproduce_trace(ctx, port):
    s = scenes.config1()
    n, iters = 3000, s.max_iterations
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    dirs = port.fibonacci(n)
    rays = rr.Rays.emit(rr.SourceConfig(s.source, n), hist_cap=iters, directions=dirs)
    recv = rr.Receiver(*s.receivers[0])
    cfg = rr.TraceConfig(max_range=s.max_range)
    parts = []
    for _ in range(iters):
        parts.append(rr.step(tree, rays, recv, cfg).captures())
        if not rays.alive.any():
            break
    got = _concat(parts)
    oc, _ = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption)).trace(
        s.source, n, [s.receivers[0][0]], [s.receivers[0][1]], iters, s.max_range)
    assert len(got) == len(oc) > 50
    for i, r in enumerate(got):
        assert r[0] == oc.ray[i] and r[1] == oc.path[i]
        assert np.array_equal(r[2], oc.point[i]) and np.array_equal(r[3], oc.dir[i])
        assert np.array_equal(r[4], oc.mult[i]) and np.array_equal(r[5], oc.history(i))


def test_brute_equals_tree_and_device_in_place(ctx):
    v, f, a = scenes.subdivided_tetrahedron(12)
    tree = rr.AccelTree(rr.TriangleMesh(v, f, a), ctx)
    src = rr.SourceConfig((0.0, 0.0, 0.0), 4096)
    recv = rr.Receiver((1e6, 1e6, 1e6), 1e-3)
    cfg = rr.TraceConfig(max_range=1e30)
    host = rr.Rays.emit(src, hist_cap=8)
    brute = rr.Rays.emit(src, hist_cap=8)
    dev = rr.Rays(*[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in
                    (host.origin, host.dir, host.mult, host.path, host.alive, host.hist, host.n_hist)])
    for _ in range(4):
        rr.step(tree, host, recv, cfg)
        rr.step(tree, brute, recv, cfg, brute=True)
        t = rr.step(tree, dev, recv, cfg)
        assert t.stats.n_captures == 0
    torch.cuda.synchronize()
    for name in ("origin", "dir", "mult", "path", "alive", "hist", "n_hist"):
        h, b, d = getattr(host, name), getattr(brute, name), getattr(dev, name).cpu().numpy()
        assert np.array_equal(h, b), name
        assert np.array_equal(h, d), name
    assert host.alive.all() and (host.n_hist == 4).all()  # closed fixture: nothing escapes
