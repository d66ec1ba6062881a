"""The reference's acceptance criteria (tests/acceptance/acceptance_main.cpp)
run on the GPU path: 1 + 2 the free-field inverse-square law and the range
cut-off (:98-157), 3 the reflecting sphere's Dirac comb (:162-234), 5 tree
traversal equal to brute force on random soups (:277-322).  Criterion 4
(shoebox against the mirror lattice) is
tests/test_gpu_facade.py::test_pipeline_shoebox_acceptance and, at C2 size,
tests/test_gpu_shoebox.py::test_c2_images_sit_on_the_lattice.  Random inputs
come from seeded numpy generators of the reference's shapes (it uses
std::mt19937)."""
import math

import numpy as np
import pytest

from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu


def test_inverse_square_law_and_range_cutoff():
    """Criteria 1 + 2: 10^6 rays in a 200 m absorbent box, receiver r = 0.36
    at six distances; direct captures follow N r^2 / (4 d^2) within 1 dB
    (3 dB below 50 expected), the derived range is exactly (r/2) sqrt(N) =
    180 m and no capture lies beyond it."""
    v, f, a = scenes.box_scene((200.0, 200.0, 200.0), absorption=1.0)
    tree = AccelTree(TriangleMesh(v, f, a))
    n, radius = 1_000_000, 0.36
    max_path = 0.0
    for d in (5.0, 10.0, 20.0, 40.0, 80.0, 160.0):
        res = rr.trace(tree, SourceConfig((5.0, 100.0, 100.0), n), Receiver((5.0 + d, 100.0, 100.0), radius),
                       TraceConfig())
        assert res.max_range == 180.0
        c = res.captures
        if len(c):
            max_path = max(max_path, float(c.path.max()))
        direct = int(np.sum(np.diff(c.hist_off) == 0))
        expected = n * radius * radius / (4.0 * d * d)
        tol = 1.0 if expected >= 50.0 else (3.0 if expected >= 5.0 else -1.0)
        if tol > 0:
            assert direct > 0 and abs(10.0 * math.log10(max(1.0, direct) / expected)) <= tol, (d, direct, expected)
    assert max_path <= 180.0


def _pulse(c, center):
    """Weighted path statistics of the captures within 0.5 m of `center`."""
    sel = (c.path >= center - 0.5) & (c.path <= center + 0.5)
    w, p = c.mult[sel, 0], c.path[sel]
    total = float(w.sum())
    if total == 0.0:
        return 0.0, 0.0, 0.0, 0.0
    mean = float((w * p).sum() / total)
    std = math.sqrt(max(0.0, float((w * p * p).sum() / total) - mean * mean))
    within = float(w[np.abs(p - center) <= 0.05].sum() / total)
    return within, mean, std, total


def _reflecting_sphere(level):
    v, f = scenes._icosphere(level)
    f4 = np.concatenate([f, np.zeros((len(f), 1), f.dtype)], 1).astype(np.int32)
    tree = AccelTree(TriangleMesh(v, f4, np.zeros((1, 8))))
    return rr.trace(tree, SourceConfig((0.0, 0.0, 0.0), 100_000), Receiver((0.0, 0.0, 0.0), 0.99),
                    TraceConfig(max_iterations=6)).captures


def test_reflecting_sphere_dirac_comb():
    """Criterion 3: from the centre of a reflecting unit icosphere, captures
    arrive in pulses at 1, 3, 5 m: 80 % of each pulse within 5 cm, spacing
    2 m to 1 %, and the coarse sphere (1 280 faces) blurs pulse 3 at least
    three times as much as the fine one (81 920)."""
    fine, coarse = _reflecting_sphere(6), _reflecting_sphere(3)
    stats = [_pulse(fine, c) for c in (1.0, 3.0, 5.0)]
    for within, _, _, energy in stats:
        assert energy > 0.0 and within >= 0.8, stats
    spacing = (stats[2][1] - stats[0][1]) / 2.0
    assert abs(spacing - 2.0) <= 0.02, spacing
    assert _pulse(coarse, 5.0)[2] >= 3.0 * stats[2][2]


@pytest.mark.parametrize("faces", [100, 1000, 10000])
def test_tree_equals_brute_force_on_soups(faces):
    """Criterion 5: 10 000 random rays through soups of 100 / 1 000 / 10 000
    random triangles: the tree traversal returns the brute-force face and
    delta (here bit for bit)."""
    rng = np.random.default_rng(424242 + faces)
    centers = rng.uniform(0.0, 10.0, (faces * 2, 3))
    tris = centers[:, None, :] + 0.4 * rng.normal(size=(faces * 2, 3, 3))
    e1, e2 = tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0]
    keep = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1) >= 1e-9
    tris = tris[keep][:faces]
    v = tris.reshape(-1, 3)
    f = np.stack([np.arange(faces) * 3, np.arange(faces) * 3 + 1, np.arange(faces) * 3 + 2,
                  np.zeros(faces, int)], 1).astype(np.int32)
    tree = AccelTree(TriangleMesh(v, f, np.zeros((1, 8))))
    o = rng.uniform(0.0, 10.0, (10000, 3))
    d = rng.normal(size=(10000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ft, dt, _ = rr.nearest_hit(tree, o, d)
    fb, db, _ = rr.nearest_hit_brute(tree, o, d)
    assert np.array_equal(ft, fb) and np.array_equal(dt, db)
    assert (ft >= 0).sum() > 100  # the sweep reaches the hit path
