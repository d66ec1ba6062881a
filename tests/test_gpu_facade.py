"""The C++ facade (include/roomray_b200.hpp) as a reference user would call
it: tests/native/facade_parity.cpp runs build_tree -> nearest_hit -> trace ->
build_image_sources -> build_pulse_trains -> synthesize on the GPU and dumps
the results, which must match the oracle: face paths, ray ids and counts exactly; positions to 1e-10;
the broadband RIR to 1e-6 of its peak.  tests/native/facade_reuse.cpp checks
that the façade's per-thread page-locked staging buffer, reused across calls
of different sizes, leaves no stale data in the artifacts."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from paper_1811_05784_b200 import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "facade_parity.cpp")
BIN = os.path.join(ROOT, "build", "facade_parity")


def compile_facade(out=BIN):
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", os.path.join(ROOT, "paper_1811_05784_b200"), "-lroomray_b200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1811_05784_b200"), "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_facade_compiles(tmp_path):
    """Header + program build warning-free against the exported ABI."""
    compile_facade(str(tmp_path / "facade_parity"))


@pytest.mark.gpu
@pytest.mark.parametrize("merge", [False, True])
def test_facade_matches_oracle(tmp_path, port, merge):
    import oracle
    exe = compile_facade(str(tmp_path / "facade_parity"))
    s = scenes.config1()
    n_rays, max_it = 4000, s.max_iterations
    (rc, rr) = s.receivers[0]
    inp = tmp_path / "in"
    out = tmp_path / "out"
    inp.mkdir()
    out.mkdir()
    s.vertices.astype(np.float64).tofile(inp / "vertices.f64")
    s.faces.astype(np.int32).tofile(inp / "faces.i32")
    s.absorption.astype(np.float64).tofile(inp / "alpha.f64")
    np.array([*s.source, *rc, rr, 343.0, s.sample_rate], np.float64).tofile(inp / "params.f64")
    r = subprocess.run([exe, str(inp), str(out), str(n_rays), str(max_it), repr(s.max_range), str(int(merge))],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout

    sc = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    tree = sc.tree()
    info = np.fromfile(out / "tree_info.i64", np.int64)
    assert info[0] == 2 * len(s.faces) - 1 and info[1] == tree.root and info[2] == tree.depth
    assert info[3] == len(s.faces)

    hits = np.fromfile(out / "hits.f64").reshape(-1, 4)
    assert np.array_equal(hits[:, 0], hits[:, 2]) and np.array_equal(hits[:, 1], hits[:, 3])

    # The facade's trace() evaluates the lattice on the device with a
    # correctly rounded sin/cos; glibc (the reference's emission) is off by
    # one ulp on ~0.3 % of the azimuths, so trajectories agree to rounding
    # (north_star: positions and delays to 1e-5 relative), face paths exactly.
    cap, st = sc.trace(s.source, n_rays, [rc], [rr], max_it, s.max_range)
    ray = np.fromfile(out / "cap_ray.i32", np.int32)
    cf = np.fromfile(out / "cap_f.f64").reshape(-1, 15)
    off = np.fromfile(out / "cap_off.i64", np.int64)
    hist = np.fromfile(out / "cap_hist.i32", np.int32)
    assert len(ray) == len(cap) > 0
    assert np.array_equal(ray, cap.ray)
    assert np.array_equal(off, cap.hist_off) and np.array_equal(hist, cap.hist[: off[-1]])
    np.testing.assert_allclose(cf[:, 0:3], cap.point, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(cf[:, 3:6], cap.dir, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(cf[:, 6], cap.path, rtol=1e-12)
    assert np.array_equal(cf[:, 7:15], cap.mult)
    assert np.mean(np.all(cf[:, 0:7] == np.c_[cap.point, cap.dir, cap.path], axis=1)) > 0.9
    stats = np.fromfile(out / "trace_stats.f64")
    assert stats[2] == st.escaped and stats[3] == st.out_of_range and stats[5] == st.ray_bounces

    ref = sc.image_sources(cap, n_rays, np.array([1.0, 20.0, 50.0, 101.325]), np.array(rc), 1e-6, merge)
    imf = np.fromfile(out / "img_f.f64").reshape(-1, 26)
    ioff = np.fromfile(out / "img_off.i64", np.int64)
    ipath = np.fromfile(out / "img_path.i32", np.int32)
    assert len(imf) == len(ref) > 0
    np.testing.assert_allclose(imf[:, 0:3], ref.pos, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(imf[:, 3], ref.dist, rtol=1e-10)
    np.testing.assert_allclose(imf[:, 4:12], ref.energy, rtol=1e-9)
    assert np.array_equal(imf[:, 12:20], ref.mult)
    assert np.array_equal(imf[:, 20], ref.ray_count) and np.array_equal(imf[:, 21], ref.order)
    assert np.array_equal(imf[:, 22], ref.has_proj)
    hp = ref.has_proj == 1
    np.testing.assert_allclose(imf[:, 23:26][hp], ref.proj[hp], rtol=1e-9, atol=1e-9)
    assert np.array_equal(ioff, ref.path_off) and np.array_equal(ipath, ref.path[: ref.path_off[-1]])

    rir = np.fromfile(out / "rir.f64")
    want = port.synthesize(ref.dist, ref.energy, 343.0, s.sample_rate)
    assert len(rir) == len(want)
    peak = np.abs(want).max()
    np.testing.assert_allclose(rir, want, rtol=0, atol=1e-6 * peak)
    fac = np.fromfile(out / "factors.f64").reshape(9, 6, 2)
    want_f = oracle.Ref().factors(ref.dist, ref.energy, 343.0) if oracle.ref_available() else None
    if want_f is not None:
        assert np.array_equal(fac[:, :, 1], want_f[:, :, 1])
        np.testing.assert_allclose(fac[:, :, 0], want_f[:, :, 0], rtol=1e-6, atol=1e-9)
    bands = np.fromfile(out / "rir_bands.f64").reshape(8, -1)
    np.testing.assert_allclose(bands.sum(0), rir, rtol=0, atol=1e-12 * peak)


# ---------------------------------------------------------------- pipeline
PIPE_SRC = os.path.join(ROOT, "tests", "native", "pipeline_run.cpp")
CONCRETE = [0.36, 0.36, 0.44, 0.31, 0.29, 0.39, 0.25, 0.25]
PODIUM = [0.4, 0.4, 0.3, 0.2, 0.17, 0.15, 0.1, 0.1]
BOX_OBJ = """# [5, 4, 3] m rectangular room, one material group per wall
v 0 0 0
v 5 0 0
v 5 4 0
v 0 4 0
v 0 0 3
v 5 0 3
v 5 4 3
v 0 4 3
usemtl concrete_block_coarse
f 1 5 8 4
usemtl hollow_wooden_podium
f 2 3 7 6
usemtl concrete_block_coarse
f 1 2 6 5
usemtl hollow_wooden_podium
f 4 8 7 3
usemtl concrete_block_coarse
f 1 4 3 2
usemtl hollow_wooden_podium
f 5 6 7 8
"""


def _pipeline_files(tmp_path, **over):
    import json
    mats = [{"name": "concrete_block_coarse", "absorption": CONCRETE},
            {"name": "hollow_wooden_podium", "absorption": PODIUM}]
    (tmp_path / "room.obj").write_text(BOX_OBJ)
    (tmp_path / "materials.json").write_text(json.dumps(mats))
    run = {"mesh": "room.obj", "materials": "materials.json", "source": {"position": [4, 2, 1.7], "ray_count": 20000},
           "receiver": {"center": [2, 2, 1.7], "radius": 0.2},
           "air": {"enabled": True, "temperature_c": 20, "relative_humidity": 50, "pressure_kpa": 101.325},
           "speed_of_sound": 343.0, "sample_rate": 44100.0, "max_iterations": 1000, "merge_coplanar": True}
    run.update(over)
    (tmp_path / "run.json").write_text(json.dumps(run))
    return tmp_path / "run.json"


def _compile_pipeline(out):
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    PIPE_SRC, "-L", os.path.join(ROOT, "paper_1811_05784_b200"), "-lroomray_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1811_05784_b200"), "-o", out], check=True)
    return out


@pytest.mark.parametrize("over,msg", [({"source": {"position": [4, 2, 1.7], "ray_count": 0}},
                                       "source.ray_count: must be >= 1"),
                                      ({"mesh": "missing.obj"}, "mesh: file does not exist"),
                                      ({"sample_rate": 8000.0}, "sample_rate: must be >= twice"),
                                      ({"air": {"temperature_c": 90}}, "air: air temperature outside")])
def test_pipeline_config_errors(tmp_path, over, msg):
    """RunConfig::validate (run_config.cpp:75-107) fails before any GPU work."""
    exe = _compile_pipeline(str(tmp_path / "pipeline_run"))
    out = tmp_path / "out"
    out.mkdir()
    r = subprocess.run([exe, str(_pipeline_files(tmp_path, **over)), str(out)], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 3 and msg in r.stdout, (r.returncode, r.stdout, r.stderr)


@pytest.mark.gpu
def test_pipeline_matches_oracle(tmp_path, port, ref):
    """run_trace_pipeline on the reference's shoebox fixture shape: images,
    RIR and factors against the reference's own stages."""
    import oracle
    exe = _compile_pipeline(str(tmp_path / "pipeline_run"))
    out = tmp_path / "out"
    out.mkdir()
    r = subprocess.run([exe, str(_pipeline_files(tmp_path)), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "pipeline ok" in r.stdout
    mesh = ref.parse_obj(BOX_OBJ, open(tmp_path / "materials.json").read())
    assert mesh["ok"] and len(mesh["faces"]) == 12
    sc = port.scene(oracle.Mesh(mesh["vertices"], mesh["faces"], mesh["absorption"]))
    cap, _ = sc.trace((4, 2, 1.7), 20000, [(2, 2, 1.7)], [0.2], 1000, 0.0)
    want = sc.image_sources(cap, 20000, np.array([1.0, 20.0, 50.0, 101.325]), np.array([2, 2, 1.7]), 1e-6, True)
    img = np.fromfile(out / "images.f64").reshape(-1, 14)
    assert len(img) == len(want) > 10
    np.testing.assert_allclose(img[:, 0:3], want.pos, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(img[:, 4:12], want.energy, rtol=1e-9)
    assert np.array_equal(img[:, 12], want.ray_count) and np.array_equal(img[:, 13], want.order)
    rir = np.fromfile(out / "rir.f64")
    w = ref.synthesize(want.dist, want.energy, 343.0, 44100.0)
    assert len(rir) == len(w)
    np.testing.assert_allclose(rir, w, rtol=0, atol=1e-6 * np.abs(w).max())
    fac = np.fromfile(out / "factors.f64").reshape(9, 6, 2)
    wf = ref.factors(want.dist, want.energy, 343.0)
    assert np.array_equal(fac[:, :, 1], wf[:, :, 1])
    np.testing.assert_allclose(fac[:, :, 0], wf[:, :, 0], rtol=1e-6, atol=1e-9)


@pytest.mark.gpu
def test_facade_step_matches_reference(tmp_path, ref):
    """emit + step() through the facade (host lattice with the C library's
    sin/cos, as emission.cpp evaluates it) reproduce the reference's own
    trace() truncated to the same iteration count bit for bit, with the
    tree and with tree == nullptr (brute force)."""
    import oracle
    src = os.path.join(ROOT, "tests", "native", "facade_step.cpp")
    exe = str(tmp_path / "facade_step")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    src, "-L", os.path.join(ROOT, "paper_1811_05784_b200"), "-lroomray_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1811_05784_b200"), "-o", exe], check=True)
    s = scenes.config1()
    n_rays, iters = 3000, 12
    (rc, rr) = s.receivers[0]
    inp, out = tmp_path / "in", tmp_path / "out"
    inp.mkdir()
    out.mkdir()
    s.vertices.astype(np.float64).tofile(inp / "vertices.f64")
    s.faces.astype(np.int32).tofile(inp / "faces.i32")
    s.absorption.astype(np.float64).tofile(inp / "alpha.f64")
    np.array([*s.source, *rc, rr], np.float64).tofile(inp / "params.f64")
    r = subprocess.run([exe, str(inp), str(out), str(n_rays), str(iters)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout

    cap, st = ref.scene(oracle.Mesh(s.vertices, s.faces, s.absorption)).trace(s.source, n_rays, rc, rr, iters, 0.0)
    assert len(cap) > 0
    for tag in ("tree", "brute"):
        ray = np.fromfile(out / f"{tag}_cap_ray.i32", np.int32)
        cf = np.fromfile(out / f"{tag}_cap_f.f64").reshape(-1, 15)
        off = np.fromfile(out / f"{tag}_cap_off.i64", np.int64)
        hist = np.fromfile(out / f"{tag}_cap_hist.i32", np.int32)
        assert len(ray) == len(cap), tag
        order = np.lexsort((cf[:, 6], ray))  # trace() sorts by (ray, path), tracer.cpp:143-147
        assert np.array_equal(ray[order], cap.ray)
        assert np.array_equal(cf[order, 0:3], cap.point) and np.array_equal(cf[order, 3:6], cap.dir)
        assert np.array_equal(cf[order, 6], cap.path) and np.array_equal(cf[order, 7:15], cap.mult)
        lens = np.diff(off)[order]
        assert np.array_equal(lens, np.diff(cap.hist_off))
        got = np.concatenate([hist[off[i]:off[i + 1]] for i in order]) if len(order) else hist[:0]
        assert np.array_equal(got, cap.hist[: cap.hist_off[-1]])
    rays_t = np.fromfile(out / "tree_rays.f64").reshape(n_rays, -1)
    rays_b = np.fromfile(out / "brute_rays.f64").reshape(n_rays, -1)
    assert np.array_equal(rays_t, rays_b)
    alive, n_hist = rays_t[:, 7] == 1, rays_t[:, 8]
    assert n_hist.max() <= iters and np.all(n_hist[alive] == iters)  # one face per surviving iteration
    assert np.all(rays_t[~alive, 6] > st.max_range) or np.all(n_hist[~alive] < iters)


@pytest.mark.gpu
def test_pipeline_shoebox_acceptance(tmp_path):
    """Acceptance criterion 4 (acceptance_main.cpp:239-272) through the C++
    facade: run_trace_pipeline on the 5x4x3 shoebox with 10^5 rays, then
    run_oracle (OracleConfig from JSON, pipeline.cpp:335-381) and compare at
    1e-9 m / 1.5 dB: no traced-only images, orders <= 2 within 1.5 dB."""
    import json
    exe = _compile_pipeline(str(tmp_path / "pipeline_run"))
    out = tmp_path / "out"
    out.mkdir()
    run = _pipeline_files(tmp_path, source={"position": [4, 2, 1.7], "ray_count": 100000})
    walls = {w: ("concrete_block_coarse" if w.endswith("0") else "hollow_wooden_podium")
             for w in ("x0", "x1", "y0", "y1", "z0", "z1")}
    (tmp_path / "oracle.json").write_text(json.dumps({
        "box": {"dimensions": [5, 4, 3]}, "materials": "materials.json", "walls": walls,
        "source": {"position": [4, 2, 1.7], "ray_count": 100000}, "receiver": {"center": [2, 2, 1.7], "radius": 0.2},
        "air": {"enabled": True, "temperature_c": 20, "relative_humidity": 50, "pressure_kpa": 101.325},
        "max_distance": 0}))
    r = subprocess.run([exe, str(run), str(out), str(tmp_path / "oracle.json")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    line = [x for x in r.stdout.splitlines() if x.startswith("acceptance4")][0]
    f = dict(kv.split("=") for kv in line.split()[1:])
    assert int(f["matched"]) > 0 and int(f["traced_only"]) == 0, line
    assert float(f["max_pos_err"]) <= 1e-9 and f["within"] == "1", line


def _upstream_layout(text):
    """The oracle's writers are built against the nlohmann 3.11.3 copy inside
    the cudnn-frontend wheel, which carries a local patch that prints integer
    arrays on one line ("[10,9]"); upstream nlohmann (the reference's vendored
    json.hpp) prints them one element per line, as the facade does.  Expand
    the patched form back to the upstream layout."""
    import re
    out = []
    pat = re.compile(r"^(\s*)(.*?)\[(-?\d+(?:,-?\d+)*)\](,?)$")
    for line in text.splitlines():
        m = pat.match(line)
        if not m or "\"" in m.group(3):
            out.append(line)
            continue
        ind, head, body, comma = m.groups()
        vals = body.split(",")
        out.append(f"{ind}{head}[")
        out += [f"{ind}  {v}{',' if i + 1 < len(vals) else ''}" for i, v in enumerate(vals)]
        out.append(f"{ind}]{comma}")
    return "\n".join(out) + "\n"


def _num_lines_equal_when_values_equal(a_text, b_text):
    """Line-by-line: a line may differ only where a number differs in value
    (so equal values are formatted identically, as nlohmann / %.17g do)."""
    import re
    b_text = _upstream_layout(b_text)
    al, bl = a_text.splitlines(), b_text.splitlines()
    assert len(al) == len(bl)
    num = re.compile(r"-?\d+(?:\.\d+)?(?:e[+-]\d+)?")
    for x, y in zip(al, bl):
        if x == y:
            continue
        nx, ny = num.findall(x), num.findall(y)
        assert num.sub("#", x) == num.sub("#", y), (x, y)
        assert any(float(p) != float(q) for p, q in zip(nx, ny)), (x, y)


@pytest.mark.gpu
def test_run_artifacts_match_the_reference_writers(tmp_path, ref):
    """`roomray trace` file set (pipeline.cpp:208-325) and the shoebox
    oracle / comparison files (:327-514), written by the facade
    (include/roomray_b200_artifacts.hpp) from GPU results, against the
    reference's own writers run on the reference pipeline: same files, same
    layout, values within the parity tolerances; equal values are formatted
    identically; two runs are byte-identical (acceptance 10)."""
    import json
    import struct
    if not hasattr(ref.L, "rref_run_artifacts"):
        pytest.skip("reference writers not built")
    exe = str(tmp_path / "artifacts_run")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "artifacts_run.cpp"), "-L",
                    os.path.join(ROOT, "paper_1811_05784_b200"), "-lroomray_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1811_05784_b200"), "-o", exe], check=True)
    run = _pipeline_files(tmp_path)
    walls = {w: ("concrete_block_coarse" if w.endswith("0") else "hollow_wooden_podium")
             for w in ("x0", "x1", "y0", "y1", "z0", "z1")}
    (tmp_path / "oracle.json").write_text(json.dumps({
        "box": {"dimensions": [5, 4, 3]}, "materials": "materials.json", "walls": walls,
        "source": {"position": [4, 2, 1.7], "ray_count": 20000}, "receiver": {"center": [2, 2, 1.7], "radius": 0.2},
        "max_distance": 0}))
    ours, ours2, theirs = tmp_path / "ours", tmp_path / "ours2", tmp_path / "ref"
    for out in (ours, ours2):
        r = subprocess.run([exe, str(run), str(out), str(tmp_path / "oracle.json")], capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
    ref.run_artifacts(run, theirs, tmp_path / "oracle.json")

    def files(d):
        return sorted(str(p.relative_to(d)) for p in d.rglob("*") if p.is_file())
    assert files(ours) == files(theirs)
    for name in ("image_sources.json", "metrics.json", "rir.wav"):  # acceptance 10
        assert (ours / name).read_bytes() == (ours2 / name).read_bytes(), name

    a, b = json.loads((ours / "image_sources.json").read_text()), json.loads((theirs / "image_sources.json").read_text())
    assert a["config"] == b["config"] and a["max_range_m"] == b["max_range_m"]
    assert len(a["images"]) == len(b["images"]) > 10
    for x, y in zip(a["images"], b["images"]):
        assert (x["order"], x["ray_count"], x["face_path"]) == (y["order"], y["ray_count"], y["face_path"])
        np.testing.assert_allclose(x["position"], y["position"], rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(x["band_energy"], y["band_energy"], rtol=1e-9)
        assert (x["projection"] is None) == (y["projection"] is None)
        if x["projection"] is not None:
            np.testing.assert_allclose(x["projection"], y["projection"], rtol=1e-9, atol=1e-9)
    _num_lines_equal_when_values_equal((ours / "image_sources.json").read_text(),
                                       (theirs / "image_sources.json").read_text())
    for csv in ("image_sources.csv", "band_trains.csv"):
        ta, tb = (ours / csv).read_text().splitlines(), (theirs / csv).read_text().splitlines()
        assert ta[0] == tb[0] and len(ta) == len(tb)
        fa = np.array([[float(v) if v else np.nan for v in line.split(",")] for line in ta[1:]])
        fb = np.array([[float(v) if v else np.nan for v in line.split(",")] for line in tb[1:]])
        np.testing.assert_allclose(fa, fb, rtol=1e-9, atol=1e-12, equal_nan=True)
        _num_lines_equal_when_values_equal((ours / csv).read_text(), (theirs / csv).read_text())
    wa, wb = (ours / "rir.wav").read_bytes(), (theirs / "rir.wav").read_bytes()
    assert wa[:44] == wb[:44] and len(wa) == len(wb)
    sa, sb = np.frombuffer(wa[44:], np.float32), np.frombuffer(wb[44:], np.float32)
    assert np.abs(sa - sb).max() <= 1e-6 * np.abs(sb).max()
    ma, mb = json.loads((ours / "metrics.json").read_text()), json.loads((theirs / "metrics.json").read_text())
    assert list(ma) == list(mb)
    for band in ma:
        for k in ma[band]:
            assert ma[band][k]["reliable"] == mb[band][k]["reliable"], (band, k)
            assert ma[band][k]["value"] == pytest.approx(mb[band][k]["value"], rel=1e-6, abs=1e-9), (band, k)
    for p in sorted(ours.glob("decay_*.csv")):
        da = np.loadtxt(p, delimiter=",", skiprows=1, ndmin=2)
        db = np.loadtxt(theirs / p.name, delimiter=",", skiprows=1, ndmin=2)
        assert da.shape == db.shape and np.array_equal(da[:, 0], db[:, 0])
        keep = db[:, 1] > -100.0  # the last events' tails cancel to rounding noise in both
        np.testing.assert_allclose(da[keep, 1], db[keep, 1], rtol=0, atol=1e-6)
    ca = [json.loads(x) for x in (ours / "captures.jsonl").read_text().splitlines()]
    cb = [json.loads(x) for x in (theirs / "captures.jsonl").read_text().splitlines()]
    assert [c["ray_index"] for c in ca] == [c["ray_index"] for c in cb]
    assert [c["face_history"] for c in ca] == [c["face_history"] for c in cb]
    np.testing.assert_allclose([c["point"] for c in ca], [c["point"] for c in cb], rtol=1e-10, atol=1e-10)
    ta, tb = json.loads((ours / "tree_stats.json").read_text()), json.loads((theirs / "tree_stats.json").read_text())
    assert [ta[k] for k in ("node_count", "leaf_count", "depth")] == [tb[k] for k in ("node_count", "leaf_count", "depth")]
    ra, rb = json.loads((ours / "run_report.json").read_text()), json.loads((theirs / "run_report.json").read_text())
    assert list(ra) == list(rb) and list(ra["timings_s"]) == list(rb["timings_s"])
    for k in ("mesh", "trace", "image_sources"):
        assert ra[k] == rb[k], k
    assert (ra["tree"]["node_count"], ra["tree"]["depth"]) == (rb["tree"]["node_count"], rb["tree"]["depth"])
    np.testing.assert_allclose(ra["air"]["alpha_db_per_m"], rb["air"]["alpha_db_per_m"], rtol=1e-14)
    # shoebox oracle files and the comparison report
    oa = (ours / "oracle" / "oracle_image_sources.json").read_text()
    ob = (theirs / "oracle" / "oracle_image_sources.json").read_text()
    ja, jb = json.loads(oa), json.loads(ob)
    assert ja["config"] == jb["config"] and len(ja["images"]) == len(jb["images"])
    for x, y in zip(ja["images"], jb["images"]):
        assert (x["position"], x["distance_m"], x["order"], x["wall_hits"]) == (
            y["position"], y["distance_m"], y["order"], y["wall_hits"])
        np.testing.assert_allclose(x["band_energy"], y["band_energy"], rtol=1e-12)
    _num_lines_equal_when_values_equal(oa, ob)
    cpa = json.loads((ours / "oracle" / "comparison.json").read_text())
    cpb = json.loads((theirs / "oracle" / "comparison.json").read_text())
    for k in ("matched_count", "unmatched_oracle_count", "unmatched_traced_count", "unmatched_oracle",
              "unmatched_traced"):
        assert cpa[k] == cpb[k], k
    assert [m["oracle_index"] for m in cpa["matched"]] == [m["oracle_index"] for m in cpb["matched"]]
    assert [m["traced_indices"] for m in cpa["matched"]] == [m["traced_indices"] for m in cpb["matched"]]


@pytest.mark.gpu
def test_facade_staging_reuse(tmp_path):
    """run_trace_pipeline on a large room, a small room, then the large room
    again: the repeated run's artifacts are byte-identical to the first."""
    exe = str(tmp_path / "facade_reuse")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "facade_reuse.cpp"), "-L",
                    os.path.join(ROOT, "paper_1811_05784_b200"), "-lroomray_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1811_05784_b200"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    words = out.stdout.split()
    assert words[0] == "ok" and int(words[1]) > 0 and int(words[2]) > 0 and int(words[3]) > 0, out.stdout
