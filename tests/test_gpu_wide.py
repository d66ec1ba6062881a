"""GPU parity of the traversal-tree choices and of two exactness edge cases.

* The binary SAH kernel on the deep configs (C3, C5 subsets) that default
  to the 8-wide compressed tree, bit for bit against the oracle.
* Grazing reflections off the floor of a room moved 3*10^4 m up, where one
  ulp of a hit coordinate is 3.6e-12 m: after a floor bounce with
  |d_z| ~ 1e-6 .. 1e-5 the reference can re-hit the floor at delta > 1e-6,
  which the coplanar-subtree cull must not skip (its threshold scales with
  the scene's coordinate magnitude, rr_trace.cu run_trace).  Caller rays
  through trace(directions=...) on every tree, against the oracle driven
  with the same rays.
* Several receivers with unequal radii and the automatic range
  (max_range <= 0): one device trace, each receiver against its own run of
  the unmodified reference (resolved_max_range per receiver,
  tracer.cpp:10-15).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh, _lib, scenes, trace

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1
TREES = [0, _lib.RR_TRACE_TREE8, _lib.RR_TRACE_TREE2]


def _captures_equal(g, o):
    assert len(g) == len(o), (len(g), len(o))
    for k in ("ray", "recv", "hist_off", "path", "point", "dir", "mult"):
        np.testing.assert_array_equal(getattr(g, k), getattr(o, k), err_msg=k)
    np.testing.assert_array_equal(g.hist, o.hist[: o.hist_off[-1]])


@pytest.mark.parametrize("cfg,stride", [("c3", 200), ("c5", 8000)])
def test_binary_tree_on_deep_configs(ctx, port, cfg, stride):
    s = scenes.CONFIGS[cfg]()
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    recvs = [Receiver(c, r) for c, r in s.receivers]
    tc = TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    src = SourceConfig(s.source, s.ray_count)
    r2 = trace(tree, src, recvs, tc, first=1, stride=stride, flags=_lib.RR_TRACE_TREE2)
    r8 = trace(tree, src, recvs, tc, first=1, stride=stride)
    oc, ost = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption)).trace(
        s.source, s.ray_count, [c for c, _ in s.receivers], [r for _, r in s.receivers], s.max_iterations,
        s.max_range, THREADS, 1, stride, 0)
    for res in (r2, r8):
        assert res.ray_bounces == ost.ray_bounces
        _captures_equal(res.captures, oc)


def _grazing_rays(n, seed):
    rng = np.random.default_rng(seed)
    ang = rng.uniform(-0.6, 0.6, n)
    dz = -rng.uniform(1e-6, 1e-5, n)
    d = np.stack([np.cos(ang), np.sin(ang), dz], 1)
    return d / np.linalg.norm(d, axis=1, keepdims=True)


@pytest.mark.parametrize("flags", TREES)
def test_grazing_floor_reflections_far_from_origin(ctx, port, flags):
    s = scenes.config1()
    off = np.array([1.0e3, -1.0e3, 3.0e4])
    v = s.vertices + off
    n = 4000
    dirs = _grazing_rays(n, 7)
    # 8 m room, floor at z = 3e4: start 10-80 um above the floor near x = 0.5
    src = tuple(np.array([0.5, 3.0, 4e-5]) + off)
    recv = (tuple(np.array([6.0, 3.0, 0.3]) + off), 0.5)
    tree = AccelTree(TriangleMesh(v, s.faces, s.absorption), ctx)
    res = trace(tree, SourceConfig(src, n), [Receiver(*recv)], TraceConfig(max_iterations=12, max_range=500.0),
                directions=dirs, flags=flags)
    oc, ost = port.scene(oracle.Mesh(v, s.faces, s.absorption)).trace(
        src, n, [recv[0]], [recv[1]], 12, 500.0, THREADS, directions=dirs)
    assert res.ray_bounces == ost.ray_bounces and res.escaped == ost.escaped
    assert len(oc) > 50
    _captures_equal(res.captures, oc)


def test_unequal_receivers_auto_range_vs_reference(ctx, ref):
    s = scenes.config1()
    n = 10_000
    recvs = [((6.0, 2.0, 1.2), 0.5), ((2.0, 4.0, 1.5), 0.2), ((4.0, 3.0, 2.0), 1.0)]
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    res = trace(tree, SourceConfig(s.source, n), [Receiver(c, r) for c, r in recvs],
                TraceConfig(max_iterations=s.max_iterations, max_range=0.0))
    rs = ref.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    g = res.captures
    total = 0
    for r, (c, rad) in enumerate(recvs):
        oc, ost = rs.trace(s.source, n, c, rad, s.max_iterations, 0.0, THREADS)
        assert ost.max_range == 0.5 * rad * np.sqrt(n)
        m = g.recv == r
        assert m.sum() == len(oc) > 0
        np.testing.assert_array_equal(g.ray[m], oc.ray)
        np.testing.assert_array_equal(g.path[m], oc.path)
        np.testing.assert_array_equal(g.point[m], oc.point)
        np.testing.assert_array_equal(g.mult[m], oc.mult)
        total += len(oc)
    assert total == len(g)
    assert res.max_range == 0.5 * 1.0 * np.sqrt(n)  # rays die past the largest range


@pytest.mark.parametrize("flags", TREES)
def test_double_sided_walls_pair_leaves(ctx, port, flags):
    """Every face duplicated with reversed winding at the next id (twins:
    same centroid, ids 2i and 2i + 1), so every leaf of the SAH tree is a
    2-face pair leaf and every closest hit is a tie broken by the face id.
    On the 8-wide tree a warp then often stashes more than 32 faces at once,
    which takes the per-lane fallback of the warp-cooperative leaf test
    (rr_trace_w8.cuh, RR_COOP)."""
    s = scenes.config1()
    f = np.asarray(s.faces)  # (v0, v1, v2, material)
    faces = np.empty((2 * len(f), f.shape[1]), dtype=f.dtype)
    faces[0::2] = f
    faces[1::2] = f
    faces[1::2, 0], faces[1::2, 2] = f[:, 2], f[:, 0]
    absorption = s.absorption
    n = 20000
    tree = AccelTree(TriangleMesh(s.vertices, faces, absorption), ctx)
    res = trace(tree, SourceConfig(s.source, n), [Receiver(*s.receivers[0])],
                TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range), flags=flags)
    oc, ost = port.scene(oracle.Mesh(s.vertices, faces, absorption)).trace(
        s.source, n, [s.receivers[0][0]], [s.receivers[0][1]], s.max_iterations, s.max_range, THREADS)
    assert res.ray_bounces == ost.ray_bounces and res.escaped == ost.escaped
    assert len(res.captures) > 0
    _captures_equal(res.captures, oc)
