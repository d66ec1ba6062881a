"""CPU: restatement (oracle/roomray_oracle.c) vs the reference itself
(oracle/_ref) on fresh seeded inputs — bit-exact.  Skipped where the
reference library was not built (no /root/reference and no prebuilt .so)."""
import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import scenes

AIR = np.array([1.0, 20.0, 50.0, 101.325])


def both(port, ref, v, f, a):
    m = oracle.Mesh(v, f, a)
    return port.scene(m), ref.scene(m)


@pytest.mark.parametrize("seed,n", [(1, 1), (2, 2), (3, 5), (4, 64), (5, 999), (6, 4096), (7, 20000)])
def test_trees(port, ref, seed, n):
    v, f, a = scenes.random_soup(seed, n, 10.0, 0.5)
    ps, rs = both(port, ref, v, f, a)
    tp, tr = ps.tree(), rs.tree()
    for k in ("left", "right", "face", "lo", "hi"):
        np.testing.assert_array_equal(getattr(tp, k), getattr(tr, k))
    assert (tp.root, tp.depth) == (tr.root, tr.depth)


def test_trees_gridded_walls(port, ref):
    """Many equal centroid coordinates: ties broken by face index."""
    s = scenes.config1()
    ps, rs = both(port, ref, s.vertices, s.faces, s.absorption)
    tp, tr = ps.tree(), rs.tree()
    for k in ("left", "right", "face"):
        np.testing.assert_array_equal(getattr(tp, k), getattr(tr, k))


@pytest.mark.parametrize("n_faces,seed", [(100, 11), (1000, 12), (10000, 13)])
def test_nearest_hit(port, ref, n_faces, seed):
    v, f, a = scenes.random_soup(seed, n_faces, 10.0, 0.4)
    ps, rs = both(port, ref, v, f, a)
    o, d = scenes.random_rays(seed + 100, 3000, 0.0, 10.0)
    for brute in (False, True):
        for x, y in zip(ps.nearest_hit(o, d, brute), rs.nearest_hit(o, d, brute)):
            np.testing.assert_array_equal(x, y)


def test_fibonacci(port, ref):
    np.testing.assert_array_equal(port.fibonacci(12345), ref.fibonacci(12345))


def _cmp_caps(a, b):
    for k in ("ray", "point", "dir", "path", "mult", "hist_off", "hist"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)


def test_trace_threads_and_subsets(port, ref):
    """Thread-count invariance (test_tracer.cpp:224-249) and the strided
    subset driver used for the CPU baseline."""
    s = scenes.config2()
    ps, rs = both(port, ref, s.vertices, s.faces, s.absorption)
    args = (s.source, s.ray_count)
    cp, sp = ps.trace(*args, [s.receivers[0][0]], [s.receivers[0][1]], 50, 686.0, 4, 5, 997, 0)
    cr, sr = rs.trace(*args, s.receivers[0][0], s.receivers[0][1], 50, 686.0, 3, 5, 997, 0)
    _cmp_caps(cp, cr)
    assert sp.ray_bounces == sr.ray_bounces
    assert (sp.iterations, sp.truncated, sp.escaped, sp.out_of_range) == (
        sr.iterations, sr.truncated, sr.escaped, sr.out_of_range)


@pytest.mark.parametrize("merge", [False, True])
def test_trace_images_open_scene(port, ref, merge):
    """Open mesh (a floor and two walls): escapes + captures on the way out."""
    v, f, a = scenes.box_scene((6, 5, 4), per_wall=np.tile(np.linspace(0.05, 0.6, 8), (6, 1)))
    keep = np.isin(f[:, 3], [0, 2, 4])
    ps, rs = both(port, ref, v, f[keep], a)
    cp, sp = ps.trace((2, 2, 1), 5000, [(4, 3, 1.5)], [0.4], 30, 0.0)
    cr, sr = rs.trace((2, 2, 1), 5000, (4, 3, 1.5), 0.4, 30, 0.0)
    _cmp_caps(cp, cr)
    assert sp.escaped == sr.escaped and sp.escaped > 0
    ip = ps.image_sources(cp, 5000, AIR, (4, 3, 1.5), 1e-6, merge)
    ir = rs.image_sources(cr, 5000, AIR, (4, 3, 1.5), 1e-6, merge)
    for k in ("pos", "dist", "energy", "mult", "ray_count", "order", "has_proj", "proj", "path_off", "path"):
        np.testing.assert_array_equal(getattr(ip, k), getattr(ir, k), err_msg=k)


def test_image_sources_c1_merge(port, ref):
    s = scenes.config1()
    ps, rs = both(port, ref, s.vertices, s.faces, s.absorption)
    c, _ = rs.trace(s.source, s.ray_count, s.receivers[0][0], s.receivers[0][1], 20, 343.0)
    for merge in (False, True):
        ip = ps.image_sources(c, s.ray_count, AIR, s.receivers[0][0], 1e-6, merge)
        ir = rs.image_sources(c, s.ray_count, AIR, s.receivers[0][0], 1e-6, merge)
        for k in ("pos", "dist", "energy", "ray_count", "order", "path", "proj"):
            np.testing.assert_array_equal(getattr(ip, k), getattr(ir, k), err_msg=k)


def test_image_sources_split_groups(port, ref):
    """split_group (image_sources.cpp:28-65): one face path whose retro
    points spread beyond tol is chained into several images
    (test_image_sources.cpp:77-83)."""
    v, f, a = scenes.box_scene((5, 4, 3))
    m = oracle.Mesh(v, f, a)
    ps, rs = port.scene(m), ref.scene(m)
    n = 7
    cap = oracle.Captures(np.zeros(n, np.int32), np.arange(n, dtype=np.int32),
                          np.array([[0, 0, 0], [5, 0, 0], [0, 0, 1e-7], [5, 0, 3e-6], [1, 1, 1], [1, 1, 1],
                                    [0, 0, 0]], float),
                          np.tile([1.0, 0, 0], (n, 1)), np.full(n, 2.0), np.ones((n, 8)),
                          np.array([0, 1, 2, 3, 4, 5, 7, 8], np.int64), np.array([3, 3, 3, 3, 3, 3, 2, 4], np.int32))
    cap.hist_off = np.array([0, 1, 2, 3, 4, 5, 6, 8], np.int64)
    cap.hist = np.array([3, 3, 3, 3, 3, 3, 2, 4], np.int32)
    ip = ps.image_sources(cap, 10, AIR, (2, 2, 1.5), 1e-6, False)
    ir = rs.image_sources(cap, 10, AIR, (2, 2, 1.5), 1e-6, False)
    assert len(ip) == len(ir) >= 3
    for k in ("pos", "dist", "energy", "ray_count", "order", "path"):
        np.testing.assert_array_equal(getattr(ip, k), getattr(ir, k), err_msg=k)


@pytest.mark.parametrize("fs", [44100.0, 48000.0])
def test_synthesize(port, ref, fs):
    d = scenes.uniform(31, 300, 0.0, 30.0)
    e = scenes.uniform(32, 2400, 0.0, 1.0).reshape(300, 8)
    for mask in (0xFF, 1, 0x80, 0x5A):
        np.testing.assert_array_equal(port.synthesize(d, e, 343.0, fs, 1023, mask),
                                      ref.synthesize(d, e, 343.0, fs, mask))
