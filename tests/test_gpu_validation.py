"""Device mesh validation (validate_faces_kernel, rr_api.cu) against the
unmodified reference's TriangleMesh::validate (geometry.cpp:47-75): the same
error kind, face index and message text, with the first failing face in
index order winning across kinds (the device reduces face*4 + kind with an
atomic minimum), on a 10^5-face mesh so the failing faces sit in different
blocks."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import AccelTree, TriangleMesh, scenes

pytestmark = pytest.mark.gpu


def _mesh():
    s = scenes.config2()
    return s.vertices.copy(), s.faces.copy(), s.absorption.copy()


def _both(ctx, ref, v, f, a):
    with pytest.raises(ValueError) as gpu:
        AccelTree(TriangleMesh(v, f, a), ctx)
    with pytest.raises(oracle.OracleError) as cpu:
        ref.scene(oracle.Mesh(v, f, a))
    return str(gpu.value), str(cpu.value)


def _degenerate(v, f, i):
    f[i, 1] = f[i, 0]  # a == b: zero area


@pytest.mark.parametrize("case", ["vertex_high", "vertex_negative", "material_high", "material_negative",
                                  "degenerate", "first_face_wins", "absorption"])
def test_validation_matches_reference(ctx, ref, case):
    v, f, a = _mesh()
    n = len(f)
    if case == "vertex_high":
        f[77_777, 2] = len(v)
    elif case == "vertex_negative":
        f[5, 0] = -1
    elif case == "material_high":
        f[40_000, 3] = len(a)
    elif case == "material_negative":
        f[n - 1, 3] = -3
    elif case == "degenerate":
        _degenerate(v, f, 63_210)
    elif case == "first_face_wins":
        _degenerate(v, f, 90_000)       # later face, other kind
        f[12_345, 3] = len(a) + 2       # the reference stops here
        f[99_999, 0] = len(v) + 9
    elif case == "absorption":
        a[1, 3] = 1.5
    g, c = _both(ctx, ref, v, f, a)
    assert g == c, (g, c)
    if case == "first_face_wins":
        assert "face 12345 references material" in g


def test_valid_mesh_passes(ctx, ref):
    v, f, a = _mesh()
    AccelTree(TriangleMesh(v, f, a), ctx)
    ref.scene(oracle.Mesh(v, f, a))
    assert np.isfinite(v).all()
