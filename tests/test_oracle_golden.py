"""CPU: the oracle restatement pinned against the reference.

(1) golden fixtures written by the UNMODIFIED reference (tests/golden/
    make_golden.py, oracle/_ref) — compared bit for bit;
(2) the known-answer tests of the reference's own suite, restated
    (tests/test_geometry.cpp, test_accel_tree.cpp, test_tracer.cpp,
    test_emission.cpp, test_image_sources.cpp, test_air_absorption.cpp,
    test_rir.cpp under /root/reference/proj/tests).
"""
import os

import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import scenes

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
AIR = np.array([1.0, 20.0, 50.0, 101.325])


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def mesh_of(g):
    return oracle.Mesh(g["vertices"], g["faces"], g["absorption"])


@pytest.mark.parametrize("name", ["tree_box", "tree_tetra4096", "tree_soup777", "tree_beads"])
def test_tree_matches_reference_fixture(port, name):
    g = gold(name)
    t = port.scene(mesh_of(g)).tree()
    for k in ("left", "right", "face", "lo", "hi"):
        np.testing.assert_array_equal(getattr(t, k), g[k])
    assert t.root == int(g["root"]) and t.depth == int(g["depth"])


def test_beads_median_split(port):
    """test_accel_tree.cpp:48-66: lower-x pair left, 7 nodes, depth 2."""
    g = gold("tree_beads")
    t = port.scene(mesh_of(g)).tree()
    assert len(t.left) == 7 and t.depth == 2
    root = t.root

    def leaves(n):
        return [t.face[n]] if t.face[n] >= 0 else leaves(t.left[n]) + leaves(t.right[n])

    assert sorted(leaves(t.left[root])) == [0, 1] and sorted(leaves(t.right[root])) == [2, 3]


@pytest.mark.parametrize("name", ["hit_soup1000", "hit_icosphere3"])
def test_nearest_hit_matches_reference_fixture(port, name):
    g = gold(name)
    sc = port.scene(mesh_of(g))
    f, d, p = sc.nearest_hit(g["origins"], g["dirs"])
    np.testing.assert_array_equal(f, g["face"])
    np.testing.assert_array_equal(d, g["delta"])
    np.testing.assert_array_equal(p, g["point"])
    bf, bd, _ = sc.nearest_hit(g["origins"], g["dirs"], brute=True)
    np.testing.assert_array_equal(bf, g["brute_face"])
    np.testing.assert_array_equal(bd, g["brute_delta"])


@pytest.mark.parametrize("name", ["trace_shoebox_fixture", "trace_c1", "trace_source_in_receiver"])
def test_trace_and_images_match_reference_fixture(port, name):
    g = gold(name)
    sc = port.scene(mesh_of(g))
    cap, st = sc.trace(g["source"], int(g["ray_count"]), [g["receiver"]], [float(g["radius"])],
                       int(g["max_iterations"]), float(g["max_range"]))
    assert st.iterations == int(g["iterations"]) and st.truncated == bool(g["truncated"])
    assert st.escaped == int(g["escaped"]) and st.out_of_range == int(g["out_of_range"])
    assert st.max_range == float(g["resolved_max_range"])
    np.testing.assert_array_equal(cap.ray, g["cap_ray"])
    np.testing.assert_array_equal(cap.point, g["cap_point"])
    np.testing.assert_array_equal(cap.dir, g["cap_dir"])
    np.testing.assert_array_equal(cap.path, g["cap_path"])
    np.testing.assert_array_equal(cap.mult, g["cap_mult"])
    np.testing.assert_array_equal(cap.hist_off, g["cap_hist_off"])
    np.testing.assert_array_equal(cap.hist, g["cap_hist"])
    im = sc.image_sources(cap, int(g["ray_count"]), AIR, g["receiver"], 1e-6, bool(g["merge"]))
    np.testing.assert_array_equal(im.pos, g["img_pos"])
    np.testing.assert_array_equal(im.dist, g["img_dist"])
    np.testing.assert_array_equal(im.ray_count, g["img_count"])
    np.testing.assert_array_equal(im.order, g["img_order"])
    np.testing.assert_array_equal(im.path, g["img_path"])
    np.testing.assert_array_equal(im.has_proj, g["img_has_proj"])
    np.testing.assert_array_equal(im.proj, g["img_proj"])
    np.testing.assert_array_equal(im.mult, g["img_mult"])
    np.testing.assert_array_equal(im.energy, g["img_energy"])


def test_source_inside_receiver_uses_exit(port):
    """test_tracer.cpp:251-269: 16 captures at 0.5, empty histories."""
    g = gold("trace_source_in_receiver")
    assert len(g["cap_ray"]) == 16
    np.testing.assert_allclose(g["cap_path"], 0.5, rtol=1e-12)
    assert (np.diff(g["cap_hist_off"]) == 0).all()


def test_rir_matches_reference_fixture(port):
    g = gold("rir_small")
    for b in range(8):
        np.testing.assert_array_equal(port.synthesize(g["dist"], g["energy"], 343.0, 48000.0, 1023, 1 << b),
                                      g["band_ir"][b])
    np.testing.assert_array_equal(port.synthesize(g["dist"], g["energy"], 343.0, 48000.0, 1023), g["broadband"])
    for b in range(8):
        np.testing.assert_array_equal(port.band_filter(b, 44100.0), g["kernels_44100"][b])


def test_air_matches_reference_fixture(port):
    g = gold("air")
    assert port.air_alpha([1, 20, 70, 101.325], 1000.0) == float(g["alpha_1k_20_70"])
    assert port.air_alpha([1, 20, 50, 101.325], 8000.0) == float(g["alpha_8k_20_50"])
    for t, h in [(20, 50), (20, 70), (10, 30)]:
        np.testing.assert_array_equal(port.air_beta([1, t, h, 101.325]), g[f"beta_{t}_{h}"])


# ---------------------------------------------------------------- known answers
def _single(a, b, c):
    return oracle.Mesh(np.array([a, b, c], float), np.array([[0, 1, 2, 0]]), np.zeros((1, 8)))


def test_triangle_known_answers(port):
    """test_geometry.cpp:48-73."""
    sc = port.scene(_single([0, 0, 0], [1, 0, 0], [0, 1, 0]))
    f, d, p = sc.nearest_hit([[0.25, 0.25, 1]], [[0, 0, -1]])
    assert f[0] == 0 and abs(d[0] - 1.0) < 1e-12 and np.linalg.norm(p[0] - [0.25, 0.25, 0]) < 1e-12
    assert sc.nearest_hit([[0.25, 0.25, 1]], [[0, 0, 1]])[0][0] == -1  # pointing away
    assert sc.nearest_hit([[2, 2, 1]], [[0, 0, -1]])[0][0] == -1  # barycentric outside
    assert sc.nearest_hit([[0.25, 0.25, -1]], [[0, 0, 1]])[0][0] == 0  # double sided
    assert sc.nearest_hit([[0.25, 0.25, 1e-7]], [[0, 0, -1]])[0][0] == -1  # self-hit guard


def test_sphere_known_answers(port):
    """test_geometry.cpp:75-86."""
    assert abs(port.intersect_sphere([0, 0, 0], [1, 0, 0], [5, 0, 0], 1.0) - 4.0) < 1e-12
    assert port.intersect_sphere([0, 0, 0], [0, 1, 0], [5, 0, 0], 1.0) is None
    assert abs(port.intersect_sphere([0, 0, 0], [0, 0, 1], [0, 0, 0], 1.0) - 1.0) < 1e-12
    assert port.intersect_sphere([10, 0, 0], [1, 0, 0], [5, 0, 0], 1.0) is None


def test_empty_mesh_is_rejected(port):
    """test_accel_tree.cpp:76-80."""
    with pytest.raises(oracle.OracleError, match="empty mesh"):
        port.scene(oracle.Mesh(np.zeros((0, 3)), np.zeros((0, 4), np.int32), np.zeros((1, 8))))


def test_mesh_validation(port):
    """test_geometry.cpp:132-152."""
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    with pytest.raises(oracle.OracleError, match="vertex out of range"):
        port.scene(oracle.Mesh(v, [[0, 17, 2, 0]], np.zeros((1, 8))))
    with pytest.raises(oracle.OracleError, match="material"):
        port.scene(oracle.Mesh(v, [[0, 1, 2, 3]], np.zeros((1, 8))))
    with pytest.raises(oracle.OracleError, match="degenerate"):
        port.scene(oracle.Mesh(np.array([[0, 0, 0], [0, 0, 0], [0, 1, 0]], float), [[0, 1, 2, 0]], np.zeros((1, 8))))
    bad = np.zeros((1, 8))
    bad[0, 3] = 1.5
    with pytest.raises(oracle.OracleError, match="absorption"):
        port.scene(oracle.Mesh(v, [[0, 1, 2, 0]], bad))


def test_one_bounce_concrete_multipliers(port):
    """test_tracer.cpp:44-63: one bounce on Table-1 concrete."""
    concrete = [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]
    v, f, a = scenes.box_scene((2, 2, 2), per_wall=[concrete] * 6)
    sc = port.scene(oracle.Mesh(v, f, a))
    # receiver just beyond the first bounce on the way back: capture at step 2
    cap, st = sc.trace([1, 1, 1], 1, [[0.5, 1, 1]], [0.01], 2, 100.0)
    # lattice ray 0 of N=1 is (1, 0, 0) (z = 0, phi = 0): hits x = 2 wall
    assert len(cap) == 1
    np.testing.assert_allclose(cap.mult[0], [0.64, 0.64, 0.56, 0.69, 0.71, 0.61, 0.75, 0.75], atol=1e-12)
    np.testing.assert_allclose(cap.path[0], 1.0 + 1.5 - 0.01, rtol=1e-12)


def test_fibonacci_known_answers(port):
    """test_emission.cpp:10-43: N=1 on the equator, unit norm, balanced."""
    d1 = port.fibonacci(1)
    assert d1[0, 2] == 0.0 and abs(np.linalg.norm(d1[0]) - 1) < 1e-12
    d = port.fibonacci(1000)
    assert np.abs(np.linalg.norm(d, axis=1) - 1).max() <= 1e-12
    assert np.linalg.norm(d.mean(axis=0)) <= 0.01


def test_air_known_answers(port):
    """test_air_absorption.cpp:25-46."""
    assert abs(port.air_alpha([1, 20, 70, 101.325], 1000.0) - 4.978e-3) <= 0.02 * 4.978e-3
    a8 = port.air_alpha([1, 20, 50, 101.325], 8000.0)
    assert abs(a8 - 0.105291) <= 0.02 * 0.105291
    beta = port.air_beta([1, 20, 50, 101.325])
    assert np.all(np.diff(beta) > 0) and np.all(beta >= 0)
    assert abs(np.exp(-beta[7] * 100) - 0.08853) <= 0.02 * 0.08853
    assert (port.air_beta([0, 20, 50, 101.325]) == 0).all()
    with pytest.raises(oracle.OracleError):
        port.air_beta([1, -30, 50, 101.325])


def test_rir_known_answers(port):
    """test_rir.cpp: event at t=0 -> causal kernel half, length 512; two
    events superpose; band kernels sum flat (+-1.5 dB, 88 Hz-5.6 kHz)."""
    e = np.zeros((1, 8))
    e[0, 4] = 1.0
    r = port.synthesize([0.0], e, 343.0, 44100.0)
    k = port.band_filter(4, 44100.0)
    assert len(r) == 512
    np.testing.assert_allclose(r, k[511:], rtol=1e-15, atol=0)
    assert len(port.synthesize(np.zeros(0), np.zeros((0, 8)), 343.0, 44100.0)) == 0
    s = sum(port.band_filter(b, 44100.0) for b in range(8))
    f = 88.0 * (5600.0 / 88.0) ** (np.arange(81) / 80.0)
    n = np.arange(1023)
    H = np.abs(np.exp(-2j * np.pi * np.outer(f, n) / 44100.0) @ s)
    assert np.abs(20 * np.log10(H)).max() <= 1.5
    with pytest.raises(oracle.OracleError):
        port.band_filter(7, 16000.0)


def test_lattice_energy_convention(port):
    """shoebox.cpp:43-116 oracle fixture: order-0 image is the source,
    E = r^2/(4 d^2) exp(-beta d)."""
    g = gold("lattice_shoebox")
    i0 = np.where(g["order"] == 0)[0]
    assert len(i0) == 1
    np.testing.assert_allclose(g["pos"][i0[0]], [4, 2, 1.7], atol=1e-12)
    d = g["dist"][i0[0]]
    beta = port.air_beta(AIR)
    np.testing.assert_allclose(g["energy"][i0[0]], 0.04 / (4 * d * d) * np.exp(-beta * d), rtol=1e-12)
