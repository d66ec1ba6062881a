"""Scene ingestion of the C++ facade (include/roomray_b200_io.hpp) against the
reference's own parse_obj / parse_material_table (obj_loader.cpp, compiled
unmodified into oracle/_ref): the shipped fixture and edge cases — fan
triangulation, negative and i/j/k indices, comments, CRLF, degenerate
faces, and every error with its kind and line number.  CPU only."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MATS = """[
  {"name": "concrete", "absorption": [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]},
  {"name": "wood", "absorption": [0.4, 0.4, 0.3, 0.2, 0.17, 0.15, 0.1, 0.1]},
  {"name": "glass\\u00e9", "absorption": [0, 0, 0, 0, 0, 0, 0, 1e-1]}
]"""

CASES = {
    "quads_and_fan": "v 0 0 0\nv 2 0 0\nv 2 1 0\nv 1 2 0\nv 0 1 0\nusemtl wood\nf 1 2 3 4 5\n",
    "negative_and_slashes": "# comment\nv 0 0 0\nv 1 0 0\nv 0 1 0\nv 0 0 1\nusemtl concrete\n"
                            "f -4/1/1 -3//2 -2/7\nusemtl wood\nf 1 2 4\nusemtl concrete\nf 1 3 4\n",
    "crlf_and_ignored": "v 0 0 0\r\nv 1 0 0\r\nvn 0 0 1\r\nv 0 1 0\r\ng grp\r\ns 1\r\nusemtl glassé\r\nf 1 2 3\r\n",
    "degenerate": "v 0 0 0\nv 1 0 0\nv 2 0 0\nv 0 1 0\nusemtl wood\nf 1 2 3\nf 1 2 4\nf 1 1 4\n",
    "err_index": "v 0 0 0\nv 1 0 0\nv 0 1 0\nusemtl wood\nf 1 2 9\n",
    "err_token": "v 0 0 0\nv 1 0 0\nv 0 1 0\nusemtl wood\nf 1 2 3x\n",
    "err_before_usemtl": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n",
    "err_short_face": "v 0 0 0\nv 1 0 0\nusemtl wood\nf 1 2\n",
    "err_vertex": "v 0 0\n",
    "err_material": "v 0 0 0\nv 1 0 0\nv 0 1 0\nusemtl marble\nf 1 2 3\n",
    "err_usemtl_empty": "v 0 0 0\nusemtl\n",
}


@pytest.fixture(scope="module")
def obj_exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("objbin") / "obj_parity")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "obj_parity.cpp"), "-o", out], check=True)
    return out


def _ours(exe, tmp_path, obj_text, mat_text):
    (tmp_path / "in.obj").write_text(obj_text, encoding="utf-8", newline="")
    (tmp_path / "m.json").write_text(mat_text, encoding="utf-8")
    out = tmp_path / "out"
    out.mkdir(exist_ok=True)
    subprocess.run([exe, str(tmp_path / "in.obj"), str(tmp_path / "m.json"), str(out)], check=True)
    status = (out / "status.txt").read_text().split("\n")
    head = status[0].split()
    if head[0] != "ok":
        return {"ok": False, "kind": head[0], "line": int(head[1]), "msg": status[1]}
    return {"ok": True, "vertices": np.fromfile(out / "vertices.f64").reshape(-1, 3),
            "faces": np.fromfile(out / "faces.i32", np.int32).reshape(-1, 4),
            "absorption": np.fromfile(out / "alpha.f64").reshape(-1, 8), "degenerate": int(head[1])}


def _same(a, b):
    assert a["ok"] == b["ok"], (a, b)
    if not a["ok"]:
        assert a["kind"] == b["kind"] and a["msg"] == b["msg"], (a, b)
        if a["kind"] == "parse":
            assert a["line"] == b["line"], (a, b)
        return
    for k in ("vertices", "faces", "absorption"):
        assert np.array_equal(a[k], b[k]), k
    assert a["degenerate"] == b["degenerate"]


@pytest.mark.parametrize("case", sorted(CASES))
def test_parse_obj_matches_reference(obj_exe, tmp_path, ref, case):
    if not getattr(ref, "has_obj", False):
        pytest.skip("reference obj_loader not built (no nlohmann/json)")
    _same(_ours(obj_exe, tmp_path, CASES[case], MATS), ref.parse_obj(CASES[case], MATS))


def test_reference_fixture(obj_exe, tmp_path, ref):
    fx = "/root/reference/proj/tests/fixtures"
    if not os.path.isdir(fx) or not getattr(ref, "has_obj", False):
        pytest.skip("reference fixtures not present")
    obj = open(os.path.join(fx, "shoebox.obj")).read()
    mats = open(os.path.join(fx, "materials.json")).read()
    ours = _ours(obj_exe, tmp_path, obj, mats)
    _same(ours, ref.parse_obj(obj, mats))
    assert len(ours["faces"]) == 12 and len(ours["absorption"]) == 2


@pytest.mark.parametrize("bad", ['{"name": "x"}', '[{"name": "x", "absorption": [0.1]}]',
                                 '[{"name": "x", "absorption": [0, 0, 0, 0, 0, 0, 0, 1.5]}]', '[1, 2'])
def test_material_table_errors(obj_exe, tmp_path, bad):
    r = _ours(obj_exe, tmp_path, "v 0 0 0\n", bad)
    assert not r["ok"] and r["kind"] == "other"
