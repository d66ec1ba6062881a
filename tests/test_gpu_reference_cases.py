"""The reference's own unit-test cases, restated against the GPU API.

Each test mirrors one TEST_CASE of the reference's suite (file:line cited)
with the same inputs and bounds, so the GPU path passes the checks a
reference user already relies on:
  tests/test_tracer.cpp (reflection, one bounce, escape, capture on exit,
  energy bookkeeping, specularity, sorted captures, order invariance, source
  inside the receiver, inverse-square law, truncation),
  tests/test_geometry.cpp (triangle and sphere examples, watertight cube),
  tests/test_accel_tree.cpp (median split, single leaf, empty mesh, perfect
  tree, balanced leaves).
The reference draws random inputs from std::mt19937; these use seeded numpy
generators of the same shape and size.
"""
import math

import numpy as np
import pytest

from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu

CONCRETE = [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]  # Table-1 concrete block, coarse


def _box(dims, alpha=0.0):
    v, f, a = scenes.box_scene(dims, absorption=alpha)
    return AccelTree(TriangleMesh(v, f, a))


def _single(a, b, c, alpha=0.0):
    v = np.array([a, b, c], np.float64)
    return AccelTree(TriangleMesh(v, np.array([[0, 1, 2, 0]], np.int32), np.full((1, 8), alpha)))


def _rays(origins, dirs, hist_cap=64):
    o = np.ascontiguousarray(np.atleast_2d(origins), np.float64)
    d = np.ascontiguousarray(np.atleast_2d(dirs), np.float64)
    n = len(o)
    return rr.Rays(o.copy(), d.copy(), np.ones((n, 8)), np.zeros(n), np.ones(n, np.int32),
                   np.zeros((n, hist_cap), np.int32), np.zeros(n, np.int32))


def _unit(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


# ---------------------------------------------------------------- test_tracer.cpp
def test_reflection_examples_and_identities():
    """test_tracer.cpp:25-42 through one step off a large z = 0 triangle."""
    tree = _single((-100, -100, 0), (100, -100, 0), (0, 200, 0))
    s = math.sqrt(2.0) / 2.0
    rng = np.random.default_rng(11)
    u = _unit(rng, 1000)
    u[:, 2] = -np.abs(u[:, 2]) - 0.05  # all head for the plane
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    dirs = np.concatenate([[[0, 0, -1], [s, 0, -s]], u])
    rays = _rays(np.tile([0.0, 0.0, 1.0], (len(dirs), 1)), dirs)
    rr.step(tree, rays, Receiver((500, 500, 500), 0.1), TraceConfig(max_range=1e3))
    r = rays.dir
    assert np.linalg.norm(r[0] - [0, 0, 1]) < 1e-15
    assert np.linalg.norm(r[1] - [s, 0, s]) < 1e-15
    n = np.array([0.0, 0.0, 1.0])  # oriented against the incident direction
    assert np.all(np.abs(np.linalg.norm(r, axis=1) - 1.0) <= 1e-12)
    assert np.all(np.abs(r @ n + dirs @ n) <= 1e-12)
    tan_r = r - np.outer(r @ n, n)
    tan_u = dirs - np.outer(dirs @ n, n)
    assert np.all(np.linalg.norm(tan_r - tan_u, axis=1) <= 1e-12)


def test_one_bounce_applies_the_per_band_wall_absorption():
    """test_tracer.cpp:44-63."""
    tree = _box((2, 2, 2), CONCRETE)
    rays = _rays([1, 1, 1], [1, 0, 0])
    rr.step(tree, rays, Receiver((1, 1, 1.5), 0.01), TraceConfig(max_range=100.0))
    expected = np.array([0.64, 0.64, 0.56, 0.69, 0.71, 0.61, 0.75, 0.75])
    assert np.all(np.abs(rays.mult[0] - expected) < 1e-12)
    assert rays.path[0] == pytest.approx(1.0)
    assert rays.n_hist[0] == 1
    assert np.linalg.norm(rays.dir[0] - [-1, 0, 0]) < 1e-15
    assert rays.alive[0] == 1


def test_ray_aimed_away_from_an_open_mesh_is_killed_without_capture():
    """test_tracer.cpp:65-81."""
    tree = _single((0, 0, 0), (1, 0, 0), (0, 1, 0))
    rays = _rays([0.2, 0.2, 1.0], [0, 0, 1])
    caps = rr.step(tree, rays, Receiver((50, 50, 50), 0.1), TraceConfig(max_range=100.0)).captures()
    assert len(caps) == 0
    assert rays.alive[0] == 0


def test_escaping_ray_can_still_be_captured_on_the_way_out():
    """test_tracer.cpp:83-100."""
    tree = _single((0, 0, 0), (1, 0, 0), (0, 1, 0))
    rays = _rays([0.2, 0.2, 1.0], [0, 0, 1])
    caps = rr.step(tree, rays, Receiver((0.2, 0.2, 5.0), 0.25), TraceConfig(max_range=100.0)).captures()
    assert len(caps) == 1
    assert caps.path[0] == pytest.approx(3.75)
    assert rays.alive[0] == 0


def test_energy_bookkeeping_in_a_fully_reflecting_box():
    """test_tracer.cpp:102-128: alpha = 0 keeps multipliers at 1; in a closed
    mesh only the range kills."""
    tree = _box((3, 4, 5))
    rays = rr.Rays.emit(rr.SourceConfig((1.5, 2, 2.5), 500), hist_cap=16)
    cfg = TraceConfig(max_range=40.0)
    for _ in range(12):
        rr.step(tree, rays, Receiver((1.0, 1.0, 1.0), 0.3), cfg)
        assert np.all(rays.mult == 1.0)
        dead = rays.alive == 0
        assert np.all(rays.path[dead] > cfg.max_range)


def test_shoebox_rays_stay_specular():
    """test_tracer.cpp:130-152."""
    tree = _box((5, 4, 3))
    rays = rr.Rays.emit(rr.SourceConfig((4, 2, 1.7), 200), hist_cap=16)
    initial = np.abs(rays.dir.copy())
    for _ in range(10):
        rr.step(tree, rays, Receiver((2, 2, 1.7), 0.2), TraceConfig(max_range=30.0))
        assert np.all(np.abs(np.abs(rays.dir) - initial) <= 1e-9)


def test_captures_are_monotone_in_path_length_and_sorted():
    """test_tracer.cpp:154-179 (the device lattice)."""
    tree = _box((5, 4, 3))
    rec = Receiver((2, 2, 1.7), 0.2)
    res = rr.trace(tree, SourceConfig((4, 2, 1.7), 3000), rec, TraceConfig())
    c = res.captures
    assert len(c) > 0
    ordered = (c.ray[1:] > c.ray[:-1]) | ((c.ray[1:] == c.ray[:-1]) & (c.path[1:] > c.path[:-1]))
    assert ordered.all()
    assert np.all(np.abs(np.linalg.norm(c.point - np.array(rec.center), axis=1) - rec.radius) <= 1e-9)
    assert np.all(c.path <= res.max_range)


def test_captures_are_independent_of_ray_processing_order():
    """test_tracer.cpp:181-218: forward and reversed spans, 8 steps."""
    tree = _box((5, 4, 3))
    rec, cfg = Receiver((2, 2, 1.7), 0.2), TraceConfig(max_range=25.0)
    n = 400
    fwd = rr.Rays.emit(rr.SourceConfig((4, 2, 1.7), n), hist_cap=16)
    rev = rr.Rays(*[np.ascontiguousarray(x[::-1]) for x in (fwd.origin, fwd.dir, fwd.mult, fwd.path, fwd.alive,
                                                             fwd.hist, fwd.n_hist)])
    a, b = [], []
    for _ in range(8):
        ca = rr.step(tree, fwd, rec, cfg).captures()
        cb = rr.step(tree, rev, rec, cfg).captures()
        a += list(zip(ca.ray.tolist(), ca.path.tolist()))
        b += list(zip((n - 1 - cb.ray).tolist(), cb.path.tolist()))
    a.sort()
    b.sort()
    assert len(a) == len(b) > 0
    for (ra, pa), (rb, pb) in zip(a, b):
        assert ra == rb and pa == pytest.approx(pb, rel=1e-12)


def test_repeated_step_is_deterministic():
    """test_tracer.cpp:220-249 compares thread counts; the GPU grid replaces
    thread_count, so the same span stepped twice must agree exactly."""
    tree = _box((5, 4, 3))
    rec = Receiver((2, 2, 1.7), 0.2)
    x = rr.Rays.emit(rr.SourceConfig((4, 2, 1.7), 4096), hist_cap=8)
    y = rr.Rays(*[np.copy(v) for v in (x.origin, x.dir, x.mult, x.path, x.alive, x.hist, x.n_hist)])
    for _ in range(5):
        ca = rr.step(tree, x, rec, TraceConfig(max_range=25.0)).captures()
        cb = rr.step(tree, y, rec, TraceConfig(max_range=25.0, thread_count=4)).captures()
        assert np.array_equal(ca.ray, cb.ray) and np.array_equal(ca.path, cb.path)


def test_direct_capture_with_the_source_inside_the_receiver_uses_the_exit():
    """test_tracer.cpp:251-269."""
    tree = _box((10, 10, 10))
    res = rr.trace(tree, SourceConfig((5, 5, 5), 16), Receiver((5, 5, 5), 0.5),
                   TraceConfig(max_iterations=1, max_range=100.0))
    c = res.captures
    assert len(c) == 16
    assert np.allclose(c.path, 0.5)
    assert np.all(np.diff(c.hist_off) == 0)


def test_free_space_inverse_square_law_at_18_m():
    """test_tracer.cpp:271-292: 10^6 rays, absorbent 200 m box, r = 0.36."""
    tree = _box((200, 200, 200), 1.0)
    res = rr.trace(tree, SourceConfig((100, 100, 100), 1_000_000), Receiver((118, 100, 100), 0.36), TraceConfig())
    assert res.max_range == pytest.approx(180.0)
    direct = int(np.sum(np.diff(res.captures.hist_off) == 0))
    expected = 1e6 * 0.36 * 0.36 / (4.0 * 18.0 * 18.0)
    assert abs(direct - expected) <= 3.0 * math.sqrt(expected)


def test_iteration_cap_flags_truncation():
    """test_tracer.cpp:294-309."""
    tree = _box((2, 2, 2))
    res = rr.trace(tree, SourceConfig((1, 1, 1), 8), Receiver((1, 1, 1), 0.1),
                   TraceConfig(max_iterations=3, max_range=1e6))
    assert res.truncated and res.iterations == 3


# ---------------------------------------------------------------- test_geometry.cpp
@pytest.mark.parametrize("brute", [False, True])
def test_triangle_intersection_axis_aligned_examples(brute):
    """test_geometry.cpp:48-73 through nearest_hit / nearest_hit_brute."""
    tree = _single((0, 0, 0), (1, 0, 0), (0, 1, 0))
    hit = rr.nearest_hit_brute if brute else rr.nearest_hit
    o = [[0.25, 0.25, 1], [0.25, 0.25, 1], [2, 2, 1], [0.25, 0.25, -1], [0.25, 0.25, 1e-7]]
    d = [[0, 0, -1], [0, 0, 1], [0, 0, -1], [0, 0, 1], [0, 0, -1]]
    face, delta, point = hit(tree, o, d)
    assert face[0] == 0 and delta[0] == pytest.approx(1.0)
    assert np.linalg.norm(point[0] - [0.25, 0.25, 0]) < 1e-12
    assert face[1] == -1  # pointing away
    assert face[2] == -1  # barycentric outside
    assert face[3] == 0   # double sided: hit from below
    assert face[4] == -1  # self-hit guard (delta <= 1e-6)


def test_sphere_intersection_examples():
    """test_geometry.cpp:75-86, through receiver captures of one step (an open
    one-face mesh far away, so every ray escapes after its sphere test)."""
    tree = _single((1000, 1000, 1000), (1001, 1000, 1000), (1000, 1001, 1000))
    cases = [((0, 0, 0), (1, 0, 0), (5, 0, 0), 4.0),   # entry
             ((0, 0, 0), (0, 1, 0), (5, 0, 0), None),  # miss
             ((0, 0, 0), (0, 0, 1), (0, 0, 0), 1.0),   # origin at the centre: exit
             ((10, 0, 0), (1, 0, 0), (5, 0, 0), None)]  # sphere behind
    for o, d, c, want in cases:
        rays = _rays(o, d)
        caps = rr.step(tree, rays, Receiver(c, 1.0), TraceConfig(max_range=100.0)).captures()
        if want is None:
            assert len(caps) == 0
        else:
            assert len(caps) == 1 and caps.path[0] == pytest.approx(want)


def test_watertight_cube_every_inside_ray_finds_one_nearest_hit():
    """test_geometry.cpp:120-131: 10 000 random directions from the centre."""
    tree = _box((2, 2, 2))
    d = _unit(np.random.default_rng(99), 10000)
    for hit in (rr.nearest_hit, rr.nearest_hit_brute):
        face, delta, _ = hit(tree, np.tile([1.0, 1.0, 1.0], (10000, 1)), d)
        assert np.all(face >= 0)
        assert np.all(delta <= math.sqrt(3.0) + 1e-12) and np.all(delta >= 1.0 - 1e-12)


# ---------------------------------------------------------------- test_accel_tree.cpp
def _beads(stations):
    v, f = [], []
    for x in stations:
        b = len(v)
        v += [(x, 0, 0), (x + 0.1, 0, 0), (x, 0.1, 0)]
        f.append((b, b + 1, b + 2, 0))
    return AccelTree(TriangleMesh(np.array(v, np.float64), np.array(f, np.int32), np.zeros((1, 8))))


def _leaves(nodes, n, depth, out):
    if nodes["face"][n] >= 0:
        out.append((int(nodes["face"][n]), depth))
        return
    for c in (nodes["left"][n], nodes["right"][n]):
        assert np.all(nodes["lo"][n] <= nodes["lo"][c]) and np.all(nodes["hi"][c] <= nodes["hi"][n])
        _leaves(nodes, c, depth + 1, out)


def test_median_split_on_the_largest_extent():
    """test_accel_tree.cpp:48-66."""
    t = _beads([0, 10, 20, 30])
    nd = t.nodes()
    assert t.leaf_count() == 4 and t.node_count() == 7 and t.depth() == 2
    root = t.root
    left, right = [], []
    _leaves(nd, nd["left"][root], 1, left)
    _leaves(nd, nd["right"][root], 1, right)
    assert sorted(f for f, _ in left) == [0, 1] and sorted(f for f, _ in right) == [2, 3]
    assert nd["hi"][nd["left"][root]][0] < nd["lo"][nd["right"][root]][0]


def test_single_face_is_a_single_leaf():
    """test_accel_tree.cpp:68-74."""
    t = _beads([5])
    assert t.node_count() == 1 and t.depth() == 0
    assert t.nodes()["face"][t.root] == 0


def test_empty_mesh_is_rejected():
    """test_accel_tree.cpp:76-80: std::invalid_argument -> ValueError."""
    with pytest.raises(ValueError):
        AccelTree(TriangleMesh(np.zeros((0, 3)), np.zeros((0, 4), np.int32), np.zeros((1, 8))))


def test_power_of_two_face_count_gives_a_perfect_tree():
    """test_accel_tree.cpp:82-90."""
    v, f, a = scenes.subdivided_tetrahedron(17)
    assert len(f) == 1 << 17
    t = AccelTree(TriangleMesh(v, f, a))
    assert t.leaf_count() == 1 << 17 and t.node_count() == 2 * (1 << 17) - 1 and t.depth() == 17


def test_leaves_partition_the_face_set_and_stay_balanced():
    """test_accel_tree.cpp:92-108 (777-face soup)."""
    v, f, a = scenes.random_soup(5150, 777, 10.0, 0.5)
    t = AccelTree(TriangleMesh(v, f, a))
    out = []
    _leaves(t.nodes(), t.root, 0, out)
    faces = sorted(x for x, _ in out)
    depths = [d for _, d in out]
    assert faces == list(range(len(f)))
    assert max(depths) - min(depths) <= 1
    assert max(depths) <= math.ceil(math.log2(len(f))) + 1


def test_one_face_scene_traces_to_completion():
    """A one-face mesh has a leaf root (accel_tree.cpp:43-46); the persistent
    tracer and step() must test it and finish (regression: a stashed-leaf
    traversal that never saw the leaf spun forever)."""
    tree = _single((0, 0, 0), (1, 0, 0), (0, 1, 0))
    res = rr.trace(tree, SourceConfig((0.2, 0.2, 1.0), 1000), Receiver((0.2, 0.2, 5.0), 0.25),
                   TraceConfig(max_range=100.0))
    assert res.iterations <= 3 and res.escaped == 1000
    assert len(res.captures) > 0


# ---------------------------------------------------------------- test_image_sources.cpp
def _images(tree, caps, receiver, total_rays=1000, air=None, merge=False):
    """caps: list of (point, dir, path, history) -> fetched image sources."""
    pts = np.array([c[0] for c in caps], np.float64)
    dirs = np.array([c[1] for c in caps], np.float64)
    paths = np.array([c[2] for c in caps], np.float64)
    dt = rr.import_captures(tree, np.arange(len(caps)), pts, dirs, paths, [c[3] for c in caps], receiver)
    return rr.build_image_sources(dt, total_rays, air or rr.AirModel.off(), rr.ClusterOptions(1e-6, merge))


def _toward(frm, to):
    d = np.asarray(to, np.float64) - np.asarray(frm, np.float64)
    return d / np.linalg.norm(d)


def test_retro_propagation_unfolds_mirrors():
    """test_image_sources.cpp:25-48: direct and first-order mirrors (walls
    x = 0, face 0, and x = 5, face 2)."""
    tree = _box((5, 4, 3))
    source, rc = np.array([4, 2, 1.7]), np.array([2, 2, 1.7])
    caps = []
    for img, hist in ((source, []), (np.array([-4, 2, 1.7]), [0]), (np.array([6, 2, 1.7]), [2])):
        d = _toward(img, rc)
        entry = rc - 0.2 * d
        caps.append((entry, d, np.linalg.norm(entry - img), hist))
    im = _images(tree, caps, Receiver(tuple(rc), 0.2))
    assert len(im) == 3
    got = {tuple(im.face_path(i)): im.position[i] for i in range(len(im))}
    assert np.linalg.norm(got[()] - source) < 1e-12
    assert np.linalg.norm(got[(0,)] - [-4, 2, 1.7]) < 1e-12
    assert np.linalg.norm(got[(2,)] - [6, 2, 1.7]) < 1e-12


def test_clustering_keys_on_the_exact_face_path():
    """test_image_sources.cpp:50-75: 250 captures of one path -> one image;
    the same retro point under another path stays split unless merged."""
    tree = _box((5, 4, 3))
    target = np.array([1.0, 2.0, 3.0])
    caps = []
    for i in range(250):
        d = np.array([1.0, 0.001 * i, 0.0])
        d /= np.linalg.norm(d)
        caps.append((target + 4.0 * d, d, 4.0, [7, 9]))
    rec = Receiver((2, 2, 1.7), 0.2)
    im = _images(tree, caps, rec)
    assert len(im) == 1 and im.ray_count[0] == 250 and im.order[0] == 2
    assert np.linalg.norm(im.position[0] - target) < 1e-12
    caps.append((target + np.array([4.0, 0, 0]), np.array([1.0, 0, 0]), 4.0, [7, 10]))
    assert len(_images(tree, caps, rec)) == 2
    merged = _images(tree, caps, rec, merge=True)
    assert len(merged) == 1 and merged.ray_count[0] == 251


def test_divergent_retro_points_split_even_with_one_path():
    """test_image_sources.cpp:77-83."""
    tree = _box((5, 4, 3))
    caps = [((0, 0, 0), (1, 0, 0), 2.0, [3]), ((5, 0, 0), (1, 0, 0), 2.0, [3])]
    assert len(_images(tree, caps, Receiver((2, 2, 1.7), 0.2))) == 2


def test_energy_attachment_follows_the_capture_units():
    """test_image_sources.cpp:85-120: n/N, exact halving, an absorbent wall,
    air absorption exp(-beta d); image 10 m from the receiver."""
    per_wall = np.zeros((6, 8))
    per_wall[0] = 1.0  # wall x0 (faces 0, 1) totally absorbent
    v, f, a = scenes.box_scene((5, 4, 3), per_wall=per_wall)
    tree = AccelTree(TriangleMesh(v, f, a))
    rec = Receiver((0, 0, 0), 0.2)
    direct = [((0, 0, 0.2), (0, 0, -1), 9.8, [])] * 25
    lossless = _images(tree, direct, rec, 1000)
    assert lossless.distance[0] == pytest.approx(10.0)
    assert np.all(np.abs(lossless.band_energy[0] - 0.025) < 1e-15)
    doubled = _images(tree, direct, rec, 2000)
    assert np.all(np.abs(lossless.band_energy[0] - 2.0 * doubled.band_energy[0]) < 1e-18)
    absorbed = _images(tree, [((0, 0, 0.2), (0, 0, -1), 9.8, [0])] * 25, rec, 1000)
    assert np.all(absorbed.band_energy[0] == 0.0)
    air = rr.AirModel()
    damped = _images(tree, direct, rec, 1000, air)
    beta = rr.air_beta_bands(air)
    assert np.all(damped.band_energy[0] <= lossless.band_energy[0])
    np.testing.assert_allclose(damped.band_energy[0], lossless.band_energy[0] * np.exp(-beta * 10.0), rtol=1e-12)


def test_projection_lands_on_the_reflecting_wall():
    """test_image_sources.cpp:122-139."""
    tree = _box((5, 4, 3))
    rc = np.array([2, 2, 1.7])
    caps = []
    for img, hist in ((np.array([-4, 2, 1.7]), [0]), (np.array([4, 2, 1.7]), [])):
        d = _toward(img, rc)
        entry = rc - 0.2 * d
        caps.append((entry, d, np.linalg.norm(entry - img), hist))
    im = _images(tree, caps, Receiver(tuple(rc), 0.2))
    by_order = {int(im.order[i]): i for i in range(len(im))}
    i1, i0 = by_order[1], by_order[0]
    assert im.has_projection[i1] == 1
    assert np.linalg.norm(im.projection[i1] - [0, 2, 1.7]) < 1e-12
    assert im.has_projection[i0] == 0


# ---------------------------------------------------------------- test_rir.cpp
def test_empty_image_set_gives_an_empty_response():
    """test_rir.cpp:37-42."""
    res = rr.synthesize(np.zeros(0), np.zeros((0, 8)), 343.0, 44100.0)
    assert len(res.samples) == 0


def test_single_event_at_t0_reproduces_the_causal_kernel_half():
    """test_rir.cpp:44-56: one unit event in band 4 at t = 0."""
    e = np.zeros((1, 8))
    e[0, 4] = 1.0
    res = rr.synthesize(np.zeros(1), e, 343.0, 44100.0)
    kernel = rr.design_band_filter(4, 44100.0)
    delay = (len(kernel) - 1) // 2
    assert len(res.samples) == delay + 1
    np.testing.assert_allclose(res.samples, kernel[delay:], rtol=1e-15, atol=0)


def test_two_identical_events_superpose_at_the_sample_offset():
    """test_rir.cpp:58-79: band-3 events of amplitude 0.7 at 1 s and 2 s."""
    fs = 44100.0
    e = np.zeros((2, 8))
    e[:, 3] = 0.49
    two = rr.synthesize(np.array([343.0, 686.0]), e, 343.0, fs).samples
    one = rr.synthesize(np.array([343.0]), e[:1], 343.0, fs).samples
    off = int(fs)
    expected = two.copy()
    expected[:] = 0.0
    expected[:len(one)] += one
    expected[off:off + len(one)] += one[:len(expected) - off]
    np.testing.assert_allclose(two, expected, rtol=1e-12, atol=1e-15)


def test_band_edges_share_crossovers_so_the_summed_bank_is_flat():
    """test_rir.cpp:81-94: summed bank within 1.5 dB over 88 Hz - 5.6 kHz."""
    fs = 44100.0
    total = sum(rr.design_band_filter(b, fs) for b in range(8))
    n = np.arange(len(total))
    for i in range(81):
        f = 88.0 * (5600.0 / 88.0) ** (i / 80.0)
        mag = abs(np.sum(total * np.exp(-2j * np.pi * f * n / fs)))
        assert abs(20.0 * math.log10(mag)) <= 1.5


def test_band_kernel_energy_against_the_brickwall_ideal():
    """test_rir.cpp:96-114."""
    fs = 44100.0
    for b, fc in enumerate([62.5, 125.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0, 8000.0]):
        k = rr.design_band_filter(b, fs)
        ratio = float(np.sum(k * k)) / (2.0 * fc * (math.sqrt(2.0) - 1.0 / math.sqrt(2.0)) / fs)
        assert (0.25 if b == 0 else 0.5) <= ratio <= 1.5


def test_sample_rate_must_cover_the_top_band_edge():
    """test_rir.cpp:116-119."""
    with pytest.raises(ValueError):
        rr.design_band_filter(7, 16000.0)
    rr.design_band_filter(7, 44100.0)


# ---------------------------------------------------------------- test_metrics.cpp
def _train_factors(band, events, c=343.0):
    """factors() of one band's pulse train, the events given as (t, a)."""
    d = np.array([t * c for t, _ in events], np.float64)
    e = np.zeros((len(events), 8))
    e[:, band] = [a * a for _, a in events]
    return rr.factors(d, e, c)


def test_two_equal_pulses_clarity_zero_definition_half_center_mid():
    """test_metrics.cpp:81-89."""
    f = _train_factors(4, [(0.0, 0.3), (0.1, 0.3)])["bands"][4]
    assert f["c80_db"][1]
    assert f["c80_db"][0] == pytest.approx(0.0, abs=1e-9)
    assert f["d50_pct"][0] == pytest.approx(50.0, abs=1e-9)
    assert f["ts_ms"][0] == pytest.approx(50.0, abs=1e-9)
    assert f["spl_db"][0] == pytest.approx(10.0 * math.log10(0.18), rel=1e-12)


def test_windows_are_measured_from_the_first_arrival():
    """test_metrics.cpp:91-99."""
    f = _train_factors(0, [(0.5, 0.3), (0.6, 0.3)])["bands"][0]
    assert f["c80_db"][0] == pytest.approx(0.0, abs=1e-9)
    assert f["d50_pct"][0] == pytest.approx(50.0, abs=1e-9)
    assert f["ts_ms"][0] == pytest.approx(50.0, abs=1e-6)


def test_a_lone_direct_pulse_has_all_energy_early():
    """test_metrics.cpp:101-110."""
    f = _train_factors(2, [(0.01, 0.5)])["bands"][2]
    assert f["d50_pct"][0] == pytest.approx(100.0)
    assert f["c80_db"][0] == pytest.approx(99.0)
    assert f["ts_ms"][0] == pytest.approx(0.0, abs=1e-12)
    assert not f["t30_s"][1]


def test_insufficient_decay_flags_t30_unreliable_but_not_the_rest():
    """test_metrics.cpp:112-121."""
    f = _train_factors(1, [(0.0, 1.0), (0.05, 0.5), (0.1, 0.25), (0.15, 0.125)])["bands"][1]
    assert not f["t30_s"][1] and f["spl_db"][1] and f["d50_pct"][1]


def test_band_factors_aggregate_the_mid_bands():
    """test_metrics.cpp:123-136."""
    c = 343.0
    d = np.array([0.0, 0.1 * c])
    e = np.full((2, 8), 0.09)
    e[:, 3] = 0.01
    out = rr.factors(d, e, c)
    assert out["mid"]["d50_pct"][0] == pytest.approx(50.0)
    spl500, spl1k = out["bands"][3]["spl_db"][0], out["bands"][4]["spl_db"][0]
    assert out["mid"]["spl_db"][0] == pytest.approx(0.5 * (spl500 + spl1k))


def test_factors_of_an_empty_or_silent_train_are_unreliable():
    """test_metrics.cpp:138-148."""
    f = rr.factors(np.zeros(0), np.zeros((0, 8)))["bands"][0]
    assert not f["spl_db"][1] and not f["t30_s"][1]
    g = _train_factors(0, [(0.1, 0.0)])["bands"][0]
    assert not g["spl_db"][1]


# ---------------------------------------------------------------- test_emission.cpp
def test_single_direction_sits_on_the_equator():
    """test_emission.cpp:10-15."""
    d = rr.fibonacci_directions(1)
    assert d.shape == (1, 3) and d[0, 2] == 0.0
    assert np.linalg.norm(d[0]) == pytest.approx(1.0, rel=1e-12)


def test_zero_rays_is_invalid():
    """test_emission.cpp:17-22 (fibonacci_directions and trace's emission)."""
    with pytest.raises(ValueError):
        rr.fibonacci_directions(0, count=0)
    with pytest.raises(ValueError):
        rr.trace(_box((2, 2, 2)), SourceConfig((1, 1, 1), 0), Receiver((1, 1, 1), 0.1), TraceConfig())


def test_lattice_is_unit_norm_and_balanced():
    """test_emission.cpp:24-33."""
    d = rr.fibonacci_directions(1000)
    assert np.all(np.abs(np.linalg.norm(d, axis=1) - 1.0) <= 1e-12)
    assert np.linalg.norm(d.mean(axis=0)) <= 0.01


def test_cap_counting_matches_solid_angle_fractions_at_one_million_points():
    """test_emission.cpp:35-52: 20 random caps over the 10^6 lattice."""
    n = 1_000_000
    d = rr.fibonacci_directions(n)
    rng = np.random.default_rng(2024)
    for _ in range(20):
        axis = _unit(rng, 1)[0]
        omega = rng.uniform(0.1, 4.0)
        inside = np.count_nonzero(d @ axis >= 1.0 - omega / (2.0 * math.pi)) / n
        expected = omega / (4.0 * math.pi)
        assert abs(inside - expected) <= 0.01 * expected


def test_emission_is_deterministic_and_matches_the_host_lattice():
    """test_emission.cpp:54-81: bit-reproducible, ray k carries lattice
    direction k; the device lattice equals the C library's to 1 ulp (the
    correctly rounded sin/cos differ from glibc on ~0.3 % of azimuths)."""
    a = rr.fibonacci_directions(4096)
    b = rr.fibonacci_directions(4096)
    assert np.array_equal(a, b)
    sub = rr.fibonacci_directions(4096, first=5, stride=7)
    assert np.array_equal(sub, a[5::7])
    host = rr.Rays.emit(rr.SourceConfig((1, 2, 3), 4096), hist_cap=1).dir
    np.testing.assert_allclose(a, host, rtol=0, atol=4e-16)
    assert np.all(np.linalg.norm(a[:4, None] - a[None, :4], axis=2)[np.triu_indices(4, 1)] > 1e-6)


# ---------------------------------------------------------------- test_air_absorption.cpp
def test_attenuation_grows_with_frequency_at_room_conditions():
    """test_air_absorption.cpp:9-17."""
    air = rr.AirModel()
    beta = rr.air_beta_bands(air)
    assert np.all(beta >= 0.0) and np.all(np.diff(beta) > 0)
    assert rr.air_alpha_db_per_m(air, 62.5) < rr.air_alpha_db_per_m(air, 8000.0)


def test_disabled_model_is_lossless():
    """test_air_absorption.cpp:19-23."""
    assert np.all(rr.air_beta_bands(rr.AirModel.off()) == 0.0)
    assert rr.air_alpha_db_per_m(rr.AirModel.off(), 1000.0) == 0.0


def test_reference_value_at_1khz_20c_70rh():
    """test_air_absorption.cpp:25-32: 4.978 dB/km within 2 %."""
    alpha = rr.air_alpha_db_per_m(rr.AirModel(relative_humidity=70.0), 1000.0)
    assert abs(alpha - 4.978e-3) <= 0.02 * 4.978e-3


def test_energy_and_level_conventions_agree():
    """test_air_absorption.cpp:34-46."""
    air = rr.AirModel()
    alpha = rr.air_alpha_db_per_m(air, 8000.0)
    beta = rr.air_beta_bands(air)[7]
    assert math.exp(-beta * 100.0) == pytest.approx(10.0 ** (-alpha * 100.0 / 10.0), rel=1e-12)
    assert abs(alpha - 0.105291) <= 0.02 * 0.105291
    assert math.exp(-beta * 100.0) == pytest.approx(0.08853, rel=0.02)


def test_condition_range_is_validated():
    """test_air_absorption.cpp:48-60."""
    for bad in (dict(temperature_c=-30.0), dict(relative_humidity=5.0), dict(pressure_kpa=200.0)):
        with pytest.raises(ValueError):
            rr.air_validate(rr.AirModel(**bad))
    rr.air_validate(rr.AirModel())


def test_triangle_intersection_agrees_with_a_direct_linear_solve():
    """test_geometry.cpp:88-118: 10 000 random triangles in [-1, 1]^3, origins
    in [-2, 2]^3, half the rays aimed near the centroid; delta against a
    linear solve of o + t d = a + u e1 + v e2 to 1e-9.  The triangles sit in
    cells 100 m apart in one mesh, so a ray's own triangle, when hit, is its
    nearest."""
    rng = np.random.default_rng(7041)
    n = 10000
    tri = rng.uniform(-1.0, 1.0, (n, 3, 3))
    area = 0.5 * np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1)
    tri = tri[area >= 1e-6]
    n = len(tri)
    cell = np.stack(np.unravel_index(np.arange(n), (22, 22, 22)), 1).astype(np.float64) * 100.0
    o = rng.uniform(-2.0, 2.0, (n, 3))
    d = _unit(rng, n)
    aimed = tri.mean(axis=1) + 0.3 * rng.uniform(-1.0, 1.0, (n, 3)) - o
    even = np.arange(n) % 2 == 0
    d[even] = aimed[even] / np.linalg.norm(aimed[even], axis=1, keepdims=True)
    v = (tri + cell[:, None, :]).reshape(-1, 3)
    f = np.stack([np.arange(n) * 3, np.arange(n) * 3 + 1, np.arange(n) * 3 + 2, np.zeros(n, int)], 1).astype(np.int32)
    tree = AccelTree(TriangleMesh(v, f, np.zeros((1, 8))))
    face, delta, point = rr.nearest_hit(tree, o + cell, d)
    # linear solve per triangle: [d, -e1, -e2] (t, u, v) = a - o
    e1, e2 = tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]
    A = np.stack([d, -e1, -e2], 2)
    sol = np.linalg.solve(A, (tri[:, 0] - o)[..., None])[..., 0]
    t, uu, vv = sol[:, 0], sol[:, 1], sol[:, 2]
    slow = (uu >= 0) & (vv >= 0) & (uu + vv <= 1) & (t > 1e-6)
    own = face == np.arange(n)
    edge = (np.abs(uu) < 1e-9) | (np.abs(vv) < 1e-9) | (np.abs(uu + vv - 1) < 1e-9) | (np.abs(t - 1e-6) < 1e-9)
    assert np.all((own == slow) | edge)  # same decision away from the boundaries
    hit = own & slow
    assert hit.sum() > 1000
    assert np.all(np.abs(delta[hit] - t[hit]) <= 1e-9 * np.maximum(1.0, np.abs(t[hit])))
    assert np.all(np.linalg.norm(point[hit] - (o + cell + delta[:, None] * d)[hit], axis=1)
                  <= 1e-9 * np.maximum(1.0, delta[hit]))
