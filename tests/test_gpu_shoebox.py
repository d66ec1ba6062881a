"""The shoebox mirror-lattice check on the device (rr_shoebox.cu) against the
reference's own enumerate_images / compare (shoebox.cpp:43-182, compiled
unmodified into oracle/_ref), and — at full C2 size, where the reference's
O(T * O) compare cannot run — the traced image sources of the GPU pipeline
against the analytic lattice (acceptance criterion 4,
acceptance_main.cpp:239-272: no traced-only images, position error <= 1e-9,
orders <= 2 within 1.5 dB).

Positions, distances, orders, wall hits and the match structure are
bit-exact; energies go through exp/log10 (CUDA vs glibc, a few ulp)."""
import numpy as np
import pytest

from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu

AIR = (1.0, 20.0, 50.0, 101.325)


def _walls(seed):
    return scenes.uniform(seed, 48, 0.02, 0.6).reshape(6, 8)


@pytest.mark.parametrize("case", [
    ((5.0, 4.0, 3.0), (4.0, 2.0, 1.7), (2.0, 2.0, 1.7), 31.6, 0.2, True),
    ((8.0, 6.0, 3.0), (2.0, 3.0, 1.5), (6.0, 2.0, 1.2), 80.0, 0.5, False),
    ((1.0, 7.0, 2.5), (0.5, 0.5, 0.5), (0.25, 6.9, 2.4), 45.0, 0.05, True),
])
def test_enumerate_matches_reference(ctx, ref, case):
    dims, src, recv, dmax, radius, air_on = case
    walls = _walls(int(dmax))
    air = rr.AirModel() if air_on else rr.AirModel.off()
    lat = rr.enumerate_images(dims, walls, src, recv, dmax, radius, air, ctx)
    got = lat.fetch()
    pos, dist, order, energy = ref.lattice(dims, walls, src, recv, dmax, radius,
                                           (1.0 if air_on else 0.0, 20.0, 50.0, 101.325))
    assert len(got) == len(dist) > 100
    np.testing.assert_array_equal(got.position, pos)
    np.testing.assert_array_equal(got.distance, dist)
    np.testing.assert_array_equal(got.order, order)
    np.testing.assert_array_equal(got.wall_hits, ref.last_lattice_hits)
    np.testing.assert_allclose(got.band_energy, energy, rtol=1e-13, atol=0)


@pytest.mark.parametrize("bad", [
    dict(dims=(0.0, 4.0, 3.0)),
    dict(src=(5.0, 2.0, 1.0)),       # on the wall, not strictly inside
    dict(recv=(2.0, -1.0, 1.0)),
    dict(dmax=0.0),
    dict(radius=-1.0),
])
def test_enumerate_errors(ctx, bad):
    a = dict(dims=(5.0, 4.0, 3.0), src=(4.0, 2.0, 1.7), recv=(2.0, 2.0, 1.7), dmax=10.0, radius=0.2)
    a.update(bad)
    with pytest.raises(ValueError):
        rr.enumerate_images(a["dims"], np.zeros((6, 8)), a["src"], a["recv"], a["dmax"], a["radius"],
                            rr.AirModel(), ctx)


def _traced_set(pos, energy, seed):
    """Traced images around the lattice: exact copies, jitter well inside and
    well outside pos_tol, split beams (several traced images on one oracle
    image), off-lattice strays."""
    rng = np.random.default_rng(seed)
    n = len(pos)
    pick = rng.integers(0, n, 3000)
    jitter = rng.choice([0.0, 1e-11, 3e-10, 5e-9], size=(3000, 1)) * rng.normal(size=(3000, 3))
    tp = pos[pick] + jitter
    te = energy[pick] * rng.uniform(0.2, 2.0, (3000, 8))
    te[::97] = 0.0  # zero energy: the 1e-300 floor
    strays = rng.uniform(-50, 50, (40, 3))
    return np.concatenate([tp, strays]), np.concatenate([te, rng.uniform(0, 1, (40, 8))])


@pytest.mark.parametrize("pos_tol", [1e-9, 1e-3, 0.0, -1.0])
def test_compare_matches_reference(ctx, ref, pos_tol):
    dims, src, recv = (5.0, 4.0, 3.0), (4.0, 2.0, 1.7), (2.0, 2.0, 1.7)
    o = rr.enumerate_images(dims, _walls(3), src, recv, 25.0, 0.2, rr.AirModel(), ctx).fetch()
    # duplicate a few oracle images: equal distances, the larger index must win
    dup = np.arange(0, len(o), 50)
    opos = np.concatenate([o.position, o.position[dup]])
    oen = np.concatenate([o.band_energy, o.band_energy[dup] * 0.5])
    oord = np.concatenate([o.order, o.order[dup]])
    tp, te = _traced_set(opos, oen, 17)
    got = rr.compare(rr.OracleImages(opos, np.zeros(len(opos)), oord, np.zeros((len(opos), 6), np.int32), oen),
                     (tp, te), pos_tol, 1.5, ctx)
    want = ref.compare(opos, oen, oord, tp, te, pos_tol, 1.5)
    for k in ("oracle_index", "order", "member_off", "members", "unmatched_oracle", "unmatched_traced",
              "position_error"):
        np.testing.assert_array_equal(getattr(got, k), want[k], err_msg=k)
    assert got.max_position_error == want["max_position_error"]
    np.testing.assert_allclose(got.energy_delta_db, want["energy_delta_db"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(got.rms_energy_error_db, want["rms_energy_error_db"], rtol=1e-12, atol=1e-12)
    if pos_tol > 0:
        assert len(got.oracle_index) > 100 and (np.diff(got.member_off) > 1).any()
    else:
        assert len(got.unmatched_traced) >= 40


def test_c2_images_sit_on_the_lattice(ctx):
    """Full C2 (100 000 triangles, 10^6 rays, 50 reflections, 686 m): every
    traced image source is a mirror-lattice image to 1e-9 m, and the low
    orders carry the analytic energy within 1.5 dB (acceptance 4)."""
    s = scenes.config2()
    rc, rad = s.receivers[0]
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    dt = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), Receiver(rc, rad),
                         TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range))
    im = rr.build_image_sources_device(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True))
    lat = rr.enumerate_images((8.0, 6.0, 3.0), s.absorption, s.source, rc, s.max_range + rad, rad,
                              rr.AirModel(), ctx)
    assert len(lat) > 5_000_000
    rep = rr.compare(lat, im, 1e-9, 1.5)
    assert im.n > 100_000 and len(rep.oracle_index) > 50_000
    assert len(rep.unmatched_traced) == 0
    assert rep.max_position_error <= 1e-9
    assert rep.energy_within(1.5, 2), np.abs(rep.energy_delta_db[rep.order <= 2]).max()
    # beams that merge_coplanar did not fold (split by range) still land on one image
    assert rep.member_off[-1] == im.n


# ---- the reference's own shoebox cases (tests/test_shoebox.cpp), restated
def _fixture(dmax, src=(4, 2, 1.7), recv=(2, 2, 1.7), walls=None):
    w = np.zeros((6, 8)) if walls is None else walls
    return rr.enumerate_images((5.0, 4.0, 3.0), w, src, recv, dmax, 0.2, rr.AirModel.off()).fetch()


def test_order1_images_are_the_six_wall_mirrors(ctx):
    """test_shoebox.cpp:23-40."""
    o = _fixture(12.0)
    got = {tuple(p) for p, k in zip(o.position.tolist(), o.order) if k == 1}
    assert got == {(-4, 2, 1.7), (6, 2, 1.7), (4, -2, 1.7), (4, 6, 1.7), (4, 2, -1.7), (4, 2, 4.3)}


def test_direct_image_is_the_source_itself(ctx):
    """test_shoebox.cpp:42-51."""
    o = _fixture(12.0)
    assert o.order[0] == 0 and np.array_equal(o.position[0], [4, 2, 1.7])
    assert o.distance[0] == pytest.approx(2.0)


def test_image_count_grows_with_the_cube_of_the_range(ctx):
    """test_shoebox.cpp:53-63."""
    assert 7.0 <= len(_fixture(40.0)) / len(_fixture(20.0)) <= 9.0


def test_wall_hit_counting_on_a_hand_unfolded_three_bounce_image(ctx):
    """test_shoebox.cpp:65-97: cell (2, -1, 0) of source (4, 2, 1.5)."""
    walls = np.repeat((0.1 * np.arange(1, 7))[:, None], 8, axis=1)
    o = _fixture(20.0, (4, 2, 1.5), (2, 2, 1.5), walls)
    i = int(np.nonzero(np.linalg.norm(o.position - [14, -2, 1.5], axis=1) < 1e-12)[0][0])
    assert o.order[i] == 3 and list(o.wall_hits[i]) == [1, 1, 1, 0, 0, 0]
    d = o.distance[i]
    want = 0.2 * 0.2 / (4.0 * d * d) * (1.0 - 0.1) * (1.0 - 0.2) * (1.0 - 0.3)
    assert o.band_energy[i, 0] == pytest.approx(want, rel=1e-12)


def test_lossless_box_follows_the_pure_inverse_square_law(ctx):
    """test_shoebox.cpp:99-108."""
    o = _fixture(30.0)
    want = 0.2 * 0.2 / (4.0 * o.distance ** 2)
    assert np.all(np.abs(o.band_energy - want[:, None]) < 1e-15)


def test_enumeration_is_sorted_and_deterministic(ctx):
    """test_shoebox.cpp:123-139 (incl. truncation independence)."""
    a, b, c = _fixture(25.0), _fixture(25.0), _fixture(35.0)
    assert np.array_equal(a.position, b.position)
    assert np.all(np.diff(a.distance) >= 0)
    assert np.array_equal(a.position, c.position[:len(a)])


def test_comparison_matches_aggregates_and_reports_misses(ctx):
    """test_shoebox.cpp:141-182 with both subcases."""
    o = _fixture(10.0)
    tp, te, = o.position[:-1].copy(), o.band_energy[:-1].copy()  # drop the last one
    te[0] *= 0.5  # split the first image into two half-energy beams
    tp, te = np.concatenate([tp, tp[:1]]), np.concatenate([te, te[:1]])
    rep = rr.compare(o, (tp, te), 1e-9, 1.5, ctx)
    assert len(rep.oracle_index) == len(o) - 1 and len(rep.unmatched_oracle) == 1
    assert len(rep.unmatched_traced) == 0 and rep.max_position_error <= 1e-12
    assert rep.energy_within(0.01, 1000)
    stray = rr.compare(o, (np.concatenate([tp, [[100, 100, 100]]]), np.concatenate([te, np.full((1, 8), 1e-6)])),
                       1e-9, 1.5, ctx)
    assert len(stray.unmatched_traced) == 1
    te2 = te.copy()
    te2[1] *= 2.0  # +3 dB
    off = rr.compare(o, (tp, te2), 1e-9, 1.5, ctx)
    assert not off.energy_within(1.5, 1000) and off.energy_within(3.2, 1000)
