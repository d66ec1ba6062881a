"""GPU parity: image sources (K5) and IR synthesis (K6/K7) vs the oracle.

Bars (BASELINE.json north_star): image-source positions and delays 1e-5
relative, per-band IR energies 1e-4 relative.  The image positions are summed
in the reference's order, so they are compared for exact equality as well;
energies go through exp() (CUDA vs glibc, <= 1 ulp apart).
"""
import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu

AIR = (1.0, 20.0, 50.0, 101.325)
CONCRETE = [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]
PODIUM = [0.4, 0.4, 0.3, 0.2, 0.17, 0.15, 0.1, 0.1]


def _run(ctx, port, v, f, a, src, n, recv, radius, max_it, max_range, merge):
    tree = AccelTree(TriangleMesh(v, f, a), ctx)
    dirs = port.fibonacci(n)
    dt = rr.trace_device(tree, SourceConfig(src, n), Receiver(recv, radius),
                         TraceConfig(max_iterations=max_it, max_range=max_range), directions=dirs)
    gi = rr.build_image_sources(dt, n, rr.AirModel(), rr.ClusterOptions(1e-6, merge))
    ps = port.scene(oracle.Mesh(v, f, a))
    oc, _ = ps.trace(src, n, [recv], [radius], max_it, max_range)
    oi = ps.image_sources(oc, n, AIR, recv, 1e-6, merge)
    return gi, oi


def _compare_images(gi, oi):
    assert len(gi) == len(oi)
    np.testing.assert_array_equal(gi.order, oi.order)
    np.testing.assert_array_equal(gi.ray_count, oi.ray_count)
    np.testing.assert_array_equal(gi.path_off, oi.path_off)
    np.testing.assert_array_equal(gi.path, oi.path)
    np.testing.assert_array_equal(gi.position, oi.pos)
    np.testing.assert_array_equal(gi.distance, oi.dist)
    np.testing.assert_array_equal(gi.band_multiplier, oi.mult)
    np.testing.assert_allclose(gi.band_energy, oi.energy, rtol=1e-12, atol=0)
    np.testing.assert_array_equal(gi.has_projection, oi.has_proj)
    np.testing.assert_array_equal(gi.projection, oi.proj)


@pytest.mark.parametrize("merge", [False, True])
def test_image_sources_shoebox_fixture(ctx, port, merge):
    v, f, a = scenes.box_scene((5, 4, 3), per_wall=[CONCRETE, PODIUM] * 3)
    gi, oi = _run(ctx, port, v, f, a, (4, 2, 1.7), 20000, (2, 2, 1.7), 0.2, 1000, 0.0, merge)
    _compare_images(gi, oi)
    assert len(gi) > 10


def test_image_sources_config1_merged(ctx, port):
    s = scenes.config1()
    gi, oi = _run(ctx, port, s.vertices, s.faces, s.absorption, s.source, s.ray_count, s.receivers[0][0],
                  s.receivers[0][1], s.max_iterations, s.max_range, True)
    _compare_images(gi, oi)


def test_image_sources_lattice_check(ctx, port):
    """tests/test_image_sources.cpp:141-189: traced shoebox images sit on the
    mirror lattice (to 1e-9) and total energy never exceeds E0."""
    v, f, a = scenes.box_scene((5, 4, 3))
    tree = AccelTree(TriangleMesh(v, f, a), ctx)
    n = 20000
    dt = rr.trace_device(tree, SourceConfig((4, 2, 1.7), n), Receiver((2, 2, 1.7), 0.2), TraceConfig())
    im = rr.build_image_sources(dt, n, rr.AirModel.off(), rr.ClusterOptions(1e-6, True))
    assert len(im) > 10
    L = np.array([5.0, 4.0, 3.0])
    s = np.array([4.0, 2.0, 1.7])
    p = im.position
    plus = np.remainder(p - s + L, 2 * L) - L
    minus = np.remainder(p + s + L, 2 * L) - L
    assert (np.minimum(np.abs(plus), np.abs(minus)) <= 1e-9).all()
    assert (im.band_energy.sum(axis=0) <= 1.0 + 1e-12).all()
    assert im.has_projection[im.order >= 1].all()


def test_synthesize_matches_reference_per_band(ctx, port):
    """Per-band IRs (one band's train populated at a time, the trick of
    tests/test_rir.cpp:44-56) and the broadband sum, 1023 taps."""
    rng_d = scenes.uniform(11, 3000, 1.0, 60.0)
    rng_e = 10.0 ** scenes.uniform(12, 3000 * 8, -8.0, 0.0).reshape(3000, 8)
    fs, c = 48000.0, 343.0
    res = rr.synthesize(rng_d, rng_e, c, fs, taps=1023)
    for b in range(8):
        ob = port.synthesize(rng_d, rng_e, c, fs, 1023, 1 << b)
        gb = res.band_ir[b]
        assert len(ob) == len(gb)
        e_ref, e_gpu = float((ob ** 2).sum()), float((gb ** 2).sum())
        assert abs(e_gpu - e_ref) <= 1e-4 * e_ref, (b, e_gpu, e_ref)
        assert np.abs(gb - ob).max() <= 1e-9 * np.abs(ob).max() + 1e-15
    full = port.synthesize(rng_d, rng_e, c, fs, 1023, 0xFF)
    assert np.abs(res.samples - full).max() <= 1e-9 * np.abs(full).max()


def test_synthesize_2048_taps_restated(ctx, port):
    d = scenes.uniform(21, 500, 1.0, 40.0)
    e = scenes.uniform(22, 500 * 8, 1e-6, 1.0).reshape(500, 8)
    res = rr.synthesize(d, e, 343.0, 48000.0, taps=2048)
    ref = port.synthesize(d, e, 343.0, 48000.0, 2048, 0xFF)
    assert len(ref) == len(res.samples)
    assert np.abs(res.samples - ref).max() <= 1e-9 * np.abs(ref).max()


def test_synthesize_edge_cases(ctx, port):
    # empty image set -> empty response (tests/test_rir.cpp:37-42)
    empty = rr.synthesize(np.zeros(0), np.zeros((0, 8)), 343.0, 44100.0)
    assert len(empty.samples) == 0
    # t = 0 event reproduces the causal kernel half (tests/test_rir.cpp:44-56)
    e = np.zeros((1, 8))
    e[0, 4] = 1.0
    r = rr.synthesize(np.zeros(1), e, 343.0, 44100.0)
    k = port.band_filter(4, 44100.0)
    assert len(r.samples) == 512
    np.testing.assert_allclose(r.samples, k[511:], rtol=1e-12, atol=1e-18)
    with pytest.raises(ValueError):
        rr.synthesize(np.array([-1.0]), np.ones((1, 8)), 343.0, 44100.0)
    with pytest.raises(ValueError):
        rr.synthesize(np.array([1.0]), np.ones((1, 8)), 0.0, 44100.0)
    with pytest.raises(ValueError):
        rr.design_band_filter(7, 16000.0)


def test_band_filter_matches_reference(ctx, port):
    for b in range(8):
        np.testing.assert_allclose(rr.design_band_filter(b, 44100.0), port.band_filter(b, 44100.0), rtol=1e-12,
                                   atol=1e-15)


@pytest.mark.parametrize("merge", [False, True])
def test_image_sources_config2_subset(ctx, port, merge):
    """Gridded 100 000-triangle room: thousands of coplanar beams per wall
    (large merge clusters, long shared path prefixes), 20 000 rays of the
    10^6 lattice, 50 reflections, against the oracle bit for bit."""
    s = scenes.config2()
    n, stride = s.ray_count, 50
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    cnt = n // stride
    dirs = port.fibonacci(n, 0, stride, cnt)
    rc, rad = s.receivers[0]
    dt = rr.trace_device(tree, SourceConfig(s.source, n), Receiver(rc, rad),
                         TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range), directions=dirs,
                         first=0, stride=stride)
    gi = rr.build_image_sources(dt, n, rr.AirModel(), rr.ClusterOptions(1e-6, merge))
    ps = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    oc, _ = ps.trace(s.source, n, [rc], [rad], s.max_iterations, s.max_range, 8, 0, stride, 0)
    oi = ps.image_sources(oc, n, AIR, rc, 1e-6, merge)
    assert len(oc) > 5000
    _compare_images(gi, oi)
    if merge:
        assert len(gi) < len(oc)  # coplanar beams did merge
