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
