"""GPU parity: device tree, closest hit and trace vs the CPU oracle.

Bar (BASELINE.json north_star): closest-hit faces bit-exact; here the fp64
parts are executed in the reference's operation order, so faces, deltas,
capture points, paths and band multipliers are compared for exact equality.
"""
import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import (AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh, nearest_hit,
                                   nearest_hit_brute, trace)
from paper_1811_05784_b200 import _lib, scenes

pytestmark = pytest.mark.gpu


def _mesh(v, f, a):
    return TriangleMesh(v, f, a), oracle.Mesh(v, f, a)


def _tree_equal(gpu: AccelTree, ot: oracle.Tree):
    g = gpu.nodes()
    assert gpu.node_count() == len(ot.left)
    assert gpu.root == ot.root
    assert gpu.depth() == ot.depth
    np.testing.assert_array_equal(g["left"], ot.left)
    np.testing.assert_array_equal(g["right"], ot.right)
    np.testing.assert_array_equal(g["face"], ot.face)
    np.testing.assert_array_equal(g["lo"], ot.lo)
    np.testing.assert_array_equal(g["hi"], ot.hi)


TREE_CASES = {
    "box": lambda: scenes.box_scene((5, 4, 3)),
    "c1": lambda: (lambda s: (s.vertices, s.faces, s.absorption))(scenes.config1()),
    "soup777": lambda: scenes.random_soup(5150, 777, 10.0, 0.5),
    "soup10000": lambda: scenes.random_soup(8080, 10000, 10.0, 0.4),
    "one_face": lambda: (np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.0]]), np.array([[0, 1, 2, 0]]), np.zeros((1, 8))),
    "three_faces": lambda: scenes.random_soup(3, 3, 2.0, 0.5),
}


@pytest.mark.parametrize("case", sorted(TREE_CASES))
def test_tree_topology_matches_build_tree(ctx, port, case):
    v, f, a = TREE_CASES[case]()
    gm, om = _mesh(v, f, a)
    _tree_equal(AccelTree(gm, ctx), port.scene(om).tree())


def test_tree_c2_100k(ctx, port):
    s = scenes.config2()
    gm, om = _mesh(s.vertices, s.faces, s.absorption)
    _tree_equal(AccelTree(gm, ctx), port.scene(om).tree())


def test_tree_perfect_power_of_two(ctx, port):
    # 2^17 faces -> 2^18 - 1 nodes, depth 17 (tests/test_accel_tree.cpp:82-90)
    v, f, a = scenes.random_soup(17, 1 << 17, 50.0, 0.3)
    f = f[: 1 << 17]
    if len(f) < (1 << 17):
        pytest.skip("soup lost degenerate faces")
    gm, om = _mesh(v, f, a)
    t = AccelTree(gm, ctx)
    assert t.node_count() == (1 << 18) - 1 and t.depth() == 17
    _tree_equal(t, port.scene(om).tree())


@pytest.mark.parametrize("n_faces,seed", [(100, 424242), (1000, 424243), (10000, 424244)])
def test_nearest_hit_matches_oracle_on_soups(ctx, port, n_faces, seed):
    """Acceptance criterion 5 (acceptance_main.cpp:277-322): tree == brute,
    0 disagreements over 10 000 rays per soup."""
    v, f, a = scenes.random_soup(seed, n_faces, 10.0, 0.4)
    gm, om = _mesh(v, f, a)
    tree = AccelTree(gm, ctx)
    o, d = scenes.random_rays(seed + 7, 10_000, 0.0, 10.0)
    gf, gd, gp = nearest_hit(tree, o, d)
    ps = port.scene(om)
    of, od, op = ps.nearest_hit(o, d)
    bf, bd, bp = ps.nearest_hit(o, d, brute=True)
    np.testing.assert_array_equal(gf, of)
    np.testing.assert_array_equal(gd, od)
    np.testing.assert_array_equal(gp, op)
    np.testing.assert_array_equal(gf, bf)
    assert (gf >= 0).sum() > n_faces // 10
    # device brute force agrees too
    hf, hd, _ = nearest_hit_brute(tree, o[:2000], d[:2000])
    np.testing.assert_array_equal(hf, bf[:2000])
    np.testing.assert_array_equal(hd, bd[:2000])


def test_nearest_hit_box_interior(ctx, port):
    """tests/test_accel_tree.cpp:129-145 shape: rays from inside a 4x3x2 box."""
    v, f, a = scenes.box_scene((4, 3, 2))
    gm, om = _mesh(v, f, a)
    tree = AccelTree(gm, ctx)
    u = scenes.uniform(31, 5000)
    o = np.stack([1 + 2 * u, np.full(5000, 1.5), np.full(5000, 1.0)], 1)
    _, d = scenes.random_rays(32, 5000, 0, 1)
    gf, gd, _ = nearest_hit(tree, o, d)
    of, od, _ = port.scene(om).nearest_hit(o, d, brute=True)
    np.testing.assert_array_equal(gf, of)
    np.testing.assert_array_equal(gd, od)
    assert (gf >= 0).all()


def _compare_captures(g, o, recv_filter=None):
    assert len(g) == len(o), (len(g), len(o))
    np.testing.assert_array_equal(g.ray, o.ray)
    np.testing.assert_array_equal(g.recv, o.recv)
    np.testing.assert_array_equal(g.hist_off, o.hist_off)
    np.testing.assert_array_equal(g.hist, o.hist)
    np.testing.assert_array_equal(g.path, o.path)
    np.testing.assert_array_equal(g.point, o.point)
    np.testing.assert_array_equal(g.dir, o.dir)
    np.testing.assert_array_equal(g.mult, o.mult)


# traversal trees: the default for the scene size, the 8-wide compressed
# tree (default from 2^18 faces), the binary SAH tree
TREES = [0, _lib.RR_TRACE_TREE8, _lib.RR_TRACE_TREE2]


def _trace_both(ctx, port, v, f, a, src, n, recvs, max_it, max_range, flags=0, **subset):
    gm, om = _mesh(v, f, a)
    tree = AccelTree(gm, ctx)
    # the device evaluates the lattice itself (glibc's sincos restated,
    # rr_sincos.cuh), so trajectories are compared bit for bit
    res = trace(tree, SourceConfig(src, n), [Receiver(c, r) for c, r in recvs],
                TraceConfig(max_iterations=max_it, max_range=max_range), flags=flags, **subset)
    oc, ost = port.scene(om).trace(src, n, [c for c, _ in recvs], [r for _, r in recvs], max_it, max_range,
                                   first=subset.get("first", 0), stride=subset.get("stride", 0),
                                   count=subset.get("count", 0))
    return res, oc, ost


@pytest.mark.parametrize("flags", TREES)
def test_trace_shoebox_fixture(ctx, port, flags):
    """The section-4.2 fixture (tests/fixtures/shoebox_run_small.json): [5,4,3]
    box, concrete/podium walls, 20 000 rays, receiver r=0.2."""
    concrete = [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]
    podium = [0.4, 0.4, 0.3, 0.2, 0.17, 0.15, 0.1, 0.1]
    v, f, a = scenes.box_scene((5, 4, 3), per_wall=[concrete, podium] * 3)
    res, oc, ost = _trace_both(ctx, port, v, f, a, (4, 2, 1.7), 20000, [((2, 2, 1.7), 0.2)], 1000, 0.0, flags)
    assert res.iterations == ost.iterations
    assert res.truncated == ost.truncated
    assert res.escaped == ost.escaped and res.out_of_range == ost.out_of_range
    assert res.max_range == ost.max_range
    assert res.ray_bounces == ost.ray_bounces
    _compare_captures(res.captures, oc)


@pytest.mark.parametrize("flags", TREES)
def test_trace_config1_full(ctx, port, flags):
    s = scenes.config1()
    res, oc, ost = _trace_both(ctx, port, s.vertices, s.faces, s.absorption, s.source, s.ray_count, s.receivers,
                               s.max_iterations, s.max_range, flags)
    assert (res.iterations, res.truncated, res.escaped, res.out_of_range) == (
        ost.iterations, ost.truncated, ost.escaped, ost.out_of_range)
    assert res.ray_bounces == ost.ray_bounces
    _compare_captures(res.captures, oc)


@pytest.mark.parametrize("flags", TREES)
def test_trace_multi_receiver_and_subset(ctx, port, flags):
    s = scenes.config2()
    recvs = [((6.0, 2.0, 1.2), 0.5), ((1.0, 1.0, 1.0), 0.3), ((4.0, 5.0, 2.5), 0.4)]
    res, oc, ost = _trace_both(ctx, port, s.vertices, s.faces, s.absorption, s.source, s.ray_count, recvs, 50,
                               686.0, flags, first=3, stride=97, count=0)
    assert res.ray_bounces == ost.ray_bounces
    _compare_captures(res.captures, oc)


@pytest.mark.parametrize("flags", TREES)
@pytest.mark.parametrize("offset,scale", [((1000.0, -2000.0, 500.0), 1.0), ((0.0, 0.0, 0.0), 1e-3),
                                          ((-3.0e4, 1.0e4, 2.0e3), 1.0), ((0.0, 0.0, 0.0), 250.0)])
def test_trace_far_and_scaled_scenes(ctx, port, offset, scale, flags):
    """The conservative fp32 box filter (eps = scale * 2^-19 of the largest
    coordinate, rr_geom.cuh) at other magnitudes: C1 moved 30 km off the
    origin, shrunk to 8 mm, blown up to 2 km — the captures stay
    bit-identical to the fp64 reference."""
    s = scenes.config1()
    v = s.vertices * scale + np.asarray(offset)
    src = tuple(np.asarray(s.source) * scale + np.asarray(offset))
    recvs = [(tuple(np.asarray(c) * scale + np.asarray(offset)), r * scale) for c, r in s.receivers]
    res, oc, ost = _trace_both(ctx, port, v, s.faces, s.absorption, src, 4000, recvs, s.max_iterations,
                               s.max_range * scale, flags)
    assert res.ray_bounces == ost.ray_bounces and len(oc) > 0
    _compare_captures(res.captures, oc)


@pytest.mark.parametrize("flags", TREES)
def test_trace_soup_interior_rays(ctx, port, flags):
    """An unstructured soup (overlapping boxes, no planes to cull) with rays
    from inside it: 20 000 rays, 30 bounces, escapes."""
    v, f, a = scenes.random_soup(424242, 20000, 10.0, 0.6)
    a = np.full_like(a, 0.05)
    res, oc, ost = _trace_both(ctx, port, v, f, a, (5.0, 5.0, 5.0), 20000, [((4.0, 6.0, 5.5), 0.7)], 30, 200.0,
                               flags)
    assert res.escaped == ost.escaped and res.ray_bounces == ost.ray_bounces
    _compare_captures(res.captures, oc)
