"""CPU oracles for the parity tests — TEST INFRASTRUCTURE ONLY.

Two ctypes-loaded libraries, built by ``oracle/Makefile``:

* ``port`` — ``oracle/roomray_oracle.c``, a plain-C restatement of the
  reference hot path (built anywhere, including the GPU box).
* ``ref``  — ``oracle/_ref/libroomray_ref.so``, the reference's own unmodified
  C++ sources compiled against a from-scratch Eigen subset (built only where
  ``/root/reference`` exists; the prebuilt .so travels with gpurun).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this package.  The product path
(``paper_1811_05784_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libroomray_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libroomray_ref.so")
REF_SRC = "/root/reference/proj"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32


def build(ref: bool | None = None) -> None:
    """Compile the port (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


@dataclass
class Mesh:
    """Plain arrays: vertices (nv,3) f64, faces (nf,4) i32 [a,b,c,material],
    absorption (nmat,8) f64 — the reference TriangleMesh (geometry.hpp:60-77)."""

    vertices: np.ndarray
    faces: np.ndarray
    absorption: np.ndarray

    def __post_init__(self):
        self.vertices = _c(self.vertices, np.float64).reshape(-1, 3)
        self.faces = _c(self.faces, np.int32).reshape(-1, 4)
        self.absorption = _c(self.absorption, np.float64).reshape(-1, 8)


@dataclass
class Tree:
    left: np.ndarray
    right: np.ndarray
    face: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    root: int
    depth: int


@dataclass
class Captures:
    recv: np.ndarray
    ray: np.ndarray
    point: np.ndarray
    dir: np.ndarray
    path: np.ndarray
    mult: np.ndarray
    hist_off: np.ndarray
    hist: np.ndarray

    def __len__(self):
        return len(self.ray)

    def history(self, i):
        return self.hist[self.hist_off[i]:self.hist_off[i + 1]]


@dataclass
class TraceStats:
    iterations: int
    truncated: bool
    escaped: int
    out_of_range: int
    max_range: float
    ray_bounces: int = -1
    sum_n_int: int = -1
    sum_n_leaf: int = -1


@dataclass
class Images:
    pos: np.ndarray
    dist: np.ndarray
    energy: np.ndarray
    mult: np.ndarray
    ray_count: np.ndarray
    order: np.ndarray
    has_proj: np.ndarray
    proj: np.ndarray
    path_off: np.ndarray
    path: np.ndarray

    def __len__(self):
        return len(self.dist)

    def face_path(self, i):
        return self.path[self.path_off[i]:self.path_off[i + 1]]


class OracleError(Exception):
    pass


# ---------------------------------------------------------------- the port
class Port:
    """ctypes view of oracle/roomray_oracle.c (the restatement)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.ro_last_error.restype = C.c_char_p
        L.ro_scene_create.restype = _vp
        L.ro_scene_create.argtypes = [_f64p, _i64, _i32p, _i64, _f64p, _i32, C.c_int]
        L.ro_scene_destroy.argtypes = [_vp]
        L.ro_tree_size.restype = _i64
        L.ro_tree_size.argtypes = [_vp, C.POINTER(_i32), C.POINTER(_i32)]
        L.ro_tree_nodes.argtypes = [_vp, _i32p, _i32p, _i32p, _f64p, _f64p]
        L.ro_face_normals.argtypes = [_vp, _f64p]
        L.ro_scene_bounds.argtypes = [_vp, _f64p, _f64p]
        L.ro_nearest_hit.argtypes = [_vp, _f64p, _f64p, _i64, C.c_int, _i32p, _f64p, _f64p, _vp, _vp]
        L.ro_intersect_sphere.argtypes = [_f64p, _f64p, _f64p, C.c_double, C.POINTER(C.c_double)]
        L.ro_fibonacci.argtypes = [_i64, _i64, _i64, _i64, _f64p]
        L.ro_trace_run.restype = _vp
        L.ro_trace_run.argtypes = [_vp, _f64p, _i64, _f64p, _f64p, _i32, _i32, C.c_double, _i32, _i64, _i64, _i64]
        L.ro_trace_run_dirs.restype = _vp
        L.ro_trace_run_dirs.argtypes = [_vp, _f64p, _i64, _f64p, _f64p, _i32, _i32, C.c_double, _i32, _i64, _i64,
                                        _i64, _vp]
        L.ro_trace_info.argtypes = [_vp, C.POINTER(_i32), C.POINTER(_i32)] + [C.POINTER(_i64)] * 2 + [
            C.POINTER(C.c_double)] + [C.POINTER(_i64)] * 5
        L.ro_trace_captures.argtypes = [_vp, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p, _i64p, _i32p]
        L.ro_trace_free.argtypes = [_vp]
        L.ro_image_sources.restype = _vp
        L.ro_image_sources.argtypes = [_vp, _i64, _i32p, _f64p, _f64p, _f64p, _f64p, _i64p, _i32p, _i64,
                                       _f64p, _f64p, C.c_double, C.c_int]
        L.ro_images_info.argtypes = [_vp, C.POINTER(_i64), C.POINTER(_i64)]
        L.ro_images_get.argtypes = [_vp, _f64p, _f64p, _f64p, _f64p, _i32p, _i32p, _i32p, _f64p, _i64p, _i32p]
        L.ro_images_free.argtypes = [_vp]
        L.ro_air_beta_bands.argtypes = [_f64p, _f64p]
        L.ro_air_alpha.restype = C.c_double
        L.ro_air_alpha.argtypes = [_f64p, C.c_double]
        L.ro_band_filter.argtypes = [C.c_int, C.c_double, C.c_int, _f64p]
        L.ro_synthesize.restype = _i64
        L.ro_synthesize.argtypes = [_i64, _f64p, _f64p, C.c_double, C.c_double, C.c_int, _i32, _vp, _i64]

    def _err(self):
        raise OracleError(self.L.ro_last_error().decode())

    # scene -------------------------------------------------------------
    def scene(self, mesh: Mesh, validate: bool = True) -> "PortScene":
        h = self.L.ro_scene_create(mesh.vertices.reshape(-1), len(mesh.vertices), mesh.faces.reshape(-1),
                                   len(mesh.faces), mesh.absorption.reshape(-1), len(mesh.absorption),
                                   int(validate))
        if not h:
            self._err()
        return PortScene(self, h, mesh)

    def fibonacci(self, n, first=0, stride=1, count=None):
        count = n if count is None else count
        out = np.empty((count, 3), np.float64)
        self.L.ro_fibonacci(n, first, stride, count, out.reshape(-1))
        return out

    def intersect_sphere(self, o, d, c, r):
        out = C.c_double()
        ok = self.L.ro_intersect_sphere(_c(o, np.float64), _c(d, np.float64), _c(c, np.float64), r, C.byref(out))
        return out.value if ok else None

    def air_beta(self, air4):
        b = np.empty(8)
        if self.L.ro_air_beta_bands(_c(air4, np.float64), b):
            self._err()
        return b

    def air_alpha(self, air4, f):
        return self.L.ro_air_alpha(_c(air4, np.float64), f)

    def band_filter(self, band, fs, taps=1023):
        out = np.empty(taps)
        if self.L.ro_band_filter(band, fs, taps, out):
            self._err()
        return out

    def synthesize(self, dist, energy, c, fs, taps=1023, band_mask=0xFF):
        dist = _c(dist, np.float64)
        energy = _c(energy, np.float64).reshape(-1)
        n = len(dist)
        length = self.L.ro_synthesize(n, dist, energy, c, fs, taps, band_mask, None, 0)
        if length < 0:
            self._err()
        out = np.zeros(length)
        if length:
            self.L.ro_synthesize(n, dist, energy, c, fs, taps, band_mask, out.ctypes.data, length)
        return out


class PortScene:
    def __init__(self, port: Port, h, mesh: Mesh):
        self.p, self.h, self.mesh = port, h, mesh

    def __del__(self):
        if getattr(self, "h", None):
            self.p.L.ro_scene_destroy(self.h)
            self.h = None

    def tree(self) -> Tree:
        root, depth = _i32(), _i32()
        n = self.p.L.ro_tree_size(self.h, C.byref(root), C.byref(depth))
        t = Tree(np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32),
                 np.empty((n, 3)), np.empty((n, 3)), root.value, depth.value)
        self.p.L.ro_tree_nodes(self.h, t.left, t.right, t.face, t.lo.reshape(-1), t.hi.reshape(-1))
        return t

    def normals(self):
        out = np.empty((len(self.mesh.faces), 3))
        self.p.L.ro_face_normals(self.h, out.reshape(-1))
        return out

    def bounds(self):
        lo, hi = np.empty(3), np.empty(3)
        self.p.L.ro_scene_bounds(self.h, lo, hi)
        return lo, hi

    def nearest_hit(self, o, d, brute=False, counts=False):
        o = _c(o, np.float64).reshape(-1, 3)
        d = _c(d, np.float64).reshape(-1, 3)
        n = len(o)
        face = np.empty(n, np.int32)
        delta = np.empty(n)
        point = np.empty((n, 3))
        ni = np.zeros(n, np.int32)
        nl = np.zeros(n, np.int32)
        self.p.L.ro_nearest_hit(self.h, o.reshape(-1), d.reshape(-1), n, int(brute), face, delta,
                                point.reshape(-1), ni.ctypes.data, nl.ctypes.data)
        if counts:
            return face, delta, point, ni, nl
        return face, delta, point

    def trace(self, src, ray_count, recv_centers, recv_radii, max_iterations=1000, max_range=0.0,
              threads=1, first=0, stride=0, count=0, directions=None):
        """trace() over the lattice subset, or over caller `directions`
        (count x 3, ray ids first + i*stride) when given."""
        rc = _c(recv_centers, np.float64).reshape(-1, 3)
        rr = _c(np.atleast_1d(recv_radii), np.float64)
        dirs = None if directions is None else _c(directions, np.float64).reshape(-1)
        h = self.p.L.ro_trace_run_dirs(self.h, _c(src, np.float64), ray_count, rc.reshape(-1), rr, len(rr),
                                       max_iterations, max_range, threads, first, stride, count,
                                       None if dirs is None else dirs.ctypes.data)
        if not h:
            self.p._err()
        try:
            it, tr = _i32(), _i32()
            esc, oor, nc, th, rb, si, sl = (_i64() for _ in range(7))
            mr = C.c_double()
            self.p.L.ro_trace_info(h, C.byref(it), C.byref(tr), C.byref(esc), C.byref(oor), C.byref(mr),
                                   C.byref(nc), C.byref(th), C.byref(rb), C.byref(si), C.byref(sl))
            n = nc.value
            cap = Captures(np.empty(n, np.int32), np.empty(n, np.int32), np.empty((n, 3)), np.empty((n, 3)),
                           np.empty(n), np.empty((n, 8)), np.empty(n + 1, np.int64),
                           np.empty(max(th.value, 1), np.int32))
            self.p.L.ro_trace_captures(h, cap.recv, cap.ray, cap.point.reshape(-1), cap.dir.reshape(-1),
                                       cap.path, cap.mult.reshape(-1), cap.hist_off, cap.hist)
            cap.hist = cap.hist[:th.value]
            st = TraceStats(it.value, bool(tr.value), esc.value, oor.value, mr.value, rb.value, si.value, sl.value)
            return cap, st
        finally:
            self.p.L.ro_trace_free(h)

    def image_sources(self, cap: Captures, total_rays, air4, recv, tol_scale=1e-6, merge_coplanar=False) -> Images:
        n = len(cap)
        h = self.p.L.ro_image_sources(self.h, n, _c(cap.ray, np.int32), _c(cap.point, np.float64).reshape(-1),
                                      _c(cap.dir, np.float64).reshape(-1), _c(cap.path, np.float64),
                                      _c(cap.mult, np.float64).reshape(-1), _c(cap.hist_off, np.int64),
                                      _c(cap.hist if len(cap.hist) else np.zeros(1), np.int32), total_rays,
                                      _c(air4, np.float64), _c(recv, np.float64), tol_scale, int(merge_coplanar))
        if not h:
            self.p._err()
        try:
            return _fetch_images(self.p.L.ro_images_info, self.p.L.ro_images_get, h)
        finally:
            self.p.L.ro_images_free(h)


def _fetch_images(info, get, h) -> Images:
    n, tp = _i64(), _i64()
    info(h, C.byref(n), C.byref(tp))
    n = n.value
    im = Images(np.empty((n, 3)), np.empty(n), np.empty((n, 8)), np.empty((n, 8)), np.empty(n, np.int32),
                np.empty(n, np.int32), np.empty(n, np.int32), np.empty((n, 3)), np.empty(n + 1, np.int64),
                np.empty(max(tp.value, 1), np.int32))
    get(h, im.pos.reshape(-1), im.dist, im.energy.reshape(-1), im.mult.reshape(-1), im.ray_count, im.order,
        im.has_proj, im.proj.reshape(-1), im.path_off, im.path)
    im.path = im.path[:tp.value]
    return im


# ---------------------------------------------------------------- the reference
class Ref:
    """ctypes view of oracle/_ref/libroomray_ref.so (unmodified reference)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError("oracle/_ref not built (needs /root/reference): " + path)
        L = C.CDLL(path)
        self.L = L
        L.rref_last_error.restype = C.c_char_p
        L.rref_scene_create.restype = _vp
        L.rref_scene_create.argtypes = [_f64p, _i64, _i32p, _i64, _f64p, _i32, C.c_int]
        L.rref_scene_destroy.argtypes = [_vp]
        L.rref_tree_size.restype = _i64
        L.rref_tree_size.argtypes = [_vp, C.POINTER(_i32), C.POINTER(_i32)]
        L.rref_tree_nodes.argtypes = [_vp, _i32p, _i32p, _i32p, _f64p, _f64p]
        L.rref_nearest_hit.argtypes = [_vp, _f64p, _f64p, _i64, C.c_int, _i32p, _f64p, _f64p]
        L.rref_intersect_sphere.argtypes = [_f64p, _f64p, _f64p, C.c_double, C.POINTER(C.c_double)]
        L.rref_fibonacci.argtypes = [C.c_int, _f64p]
        if hasattr(L, "rref_run_artifacts"):
            L.rref_run_artifacts.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
        L.rref_bench_row.restype = C.c_double
        L.rref_bench_row.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(_i32)]
        L.rref_trace.restype = _vp
        L.rref_trace.argtypes = [_vp, _f64p, _i32, _f64p, C.c_double, _i32, C.c_double, _i32, _i64, _i64, _i64]
        L.rref_trace_info.argtypes = [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i64),
                                      C.POINTER(C.c_double), C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]
        L.rref_trace_captures.argtypes = [_vp, _i32p, _f64p, _f64p, _f64p, _f64p, _i64p, _i32p]
        L.rref_trace_free.argtypes = [_vp]
        L.rref_image_sources.restype = _vp
        L.rref_image_sources.argtypes = [_vp, _i64, _i32p, _f64p, _f64p, _f64p, _f64p, _i64p, _i32p, _i32,
                                         _f64p, _f64p, C.c_double, C.c_int]
        L.rref_images_info.argtypes = [_vp, C.POINTER(_i64), C.POINTER(_i64)]
        L.rref_images_get.argtypes = [_vp, _f64p, _f64p, _f64p, _f64p, _i32p, _i32p, _i32p, _f64p, _i64p, _i32p]
        L.rref_images_free.argtypes = [_vp]
        L.rref_air_beta_bands.argtypes = [_f64p, _f64p]
        L.rref_air_alpha.restype = C.c_double
        L.rref_air_alpha.argtypes = [_f64p, C.c_double]
        L.rref_band_filter.argtypes = [C.c_int, C.c_double, _f64p]
        self.has_obj = hasattr(L, "rref_parse_obj")
        if self.has_obj:
            L.rref_parse_obj.restype = C.c_int
            L.rref_parse_obj.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(_vp), C.POINTER(_i32)]
            L.rref_obj_info.argtypes = [_vp] + [C.POINTER(_i64)] * 4
            L.rref_obj_get.argtypes = [_vp, _f64p, _i32p, _f64p]
            L.rref_obj_free.argtypes = [_vp]
        L.rref_factors.restype = C.c_int
        L.rref_factors.argtypes = [_i64, _f64p, _f64p, C.c_double, _f64p]
        L.rref_synthesize.restype = _i64
        L.rref_synthesize.argtypes = [_i64, _f64p, _f64p, C.c_double, C.c_double, _i32, _vp, _i64]
        L.rref_lattice.restype = _vp
        L.rref_lattice.argtypes = [_f64p, _f64p, _f64p, _f64p, C.c_double, C.c_double, _f64p, C.POINTER(_i64)]
        L.rref_lattice_get.argtypes = [_vp, _f64p, _f64p, _i32p, _f64p]
        L.rref_lattice_free.argtypes = [_vp]
        L.rref_lattice_hits.argtypes = [_vp, _i32p]
        L.rref_compare.restype = _vp
        L.rref_compare.argtypes = [_i64, _f64p, _f64p, _i32p, _i64, _f64p, _f64p, C.c_double, C.c_double, _i64p,
                                   C.POINTER(C.c_double), _f64p]
        L.rref_compare_get.argtypes = [_vp, _i32p, _f64p, _i32p, _f64p, _i64p, _i32p, _i32p, _i32p]
        L.rref_compare_free.argtypes = [_vp]
        L.rref_mesh_gen.restype = _vp
        L.rref_mesh_gen.argtypes = [C.c_int, _f64p, C.c_int, C.POINTER(_i64), C.POINTER(_i64)]
        L.rref_mesh_get.argtypes = [_vp, _f64p, _i32p]
        L.rref_mesh_free.argtypes = [_vp]
        L.rref_hardware_threads.restype = C.c_int
        L.rref_empty_tree_throws.restype = C.c_int

    def _err(self):
        raise OracleError(self.L.rref_last_error().decode())

    def scene(self, mesh: Mesh, validate: bool = True) -> "RefScene":
        h = self.L.rref_scene_create(mesh.vertices.reshape(-1), len(mesh.vertices), mesh.faces.reshape(-1),
                                     len(mesh.faces), mesh.absorption.reshape(-1), len(mesh.absorption),
                                     int(validate))
        if not h:
            self._err()
        return RefScene(self, h, mesh)

    def run_artifacts(self, run_json, out_dir, oracle_json=""):
        """The reference's run_trace_pipeline + write_run_artifacts (and the
        shoebox oracle files with oracle_json) into out_dir."""
        if self.L.rref_run_artifacts(str(run_json).encode(), str(out_dir).encode(), str(oracle_json).encode()):
            self._err()

    def bench_row(self, k, with_tree=True, threads=1, min_elapsed=0.25, max_repeats=50):
        """The reference's complexity-benchmark row (bench.cpp:26-46, 71-102):
        (seconds per step() iteration, build seconds, tree depth)."""
        b, d = C.c_double(), _i32()
        t = self.L.rref_bench_row(k, int(with_tree), threads, min_elapsed, max_repeats, C.byref(b), C.byref(d))
        if t < 0:
            self._err()
        return t, b.value, d.value

    def fibonacci(self, n):
        out = np.empty((n, 3))
        self.L.rref_fibonacci(n, out.reshape(-1))
        return out

    def intersect_sphere(self, o, d, c, r):
        out = C.c_double()
        ok = self.L.rref_intersect_sphere(_c(o, np.float64), _c(d, np.float64), _c(c, np.float64), r,
                                          C.byref(out))
        return out.value if ok else None

    def air_beta(self, air4):
        b = np.empty(8)
        self.L.rref_air_beta_bands(_c(air4, np.float64), b)
        return b

    def air_alpha(self, air4, f):
        return self.L.rref_air_alpha(_c(air4, np.float64), f)

    def band_filter(self, band, fs):
        out = np.empty(1023)
        if self.L.rref_band_filter(band, fs, out):
            self._err()
        return out

    def synthesize(self, dist, energy, c, fs, band_mask=0xFF):
        dist = _c(dist, np.float64)
        energy = _c(energy, np.float64).reshape(-1)
        n = len(dist)
        length = self.L.rref_synthesize(n, dist, energy, c, fs, band_mask, None, 0)
        if length < 0:
            self._err()
        out = np.zeros(length)
        if length:
            self.L.rref_synthesize(n, dist, energy, c, fs, band_mask, out.ctypes.data, length)
        return out

    def parse_obj(self, obj_text: str, mat_json: str) -> dict:
        """parse_material_table + parse_obj (obj_loader.cpp:25-152): {"ok": True,
        vertices, faces, absorption, degenerate} or {"ok": False, "kind":
        "parse" | "material" | "other", "line", "msg"}."""
        h, line = _vp(), _i32()
        rc = self.L.rref_parse_obj(obj_text.encode(), mat_json.encode(), C.byref(h), C.byref(line))
        if rc:
            return {"ok": False, "kind": {1: "parse", 2: "material"}.get(rc, "other"), "line": line.value,
                    "msg": self.L.rref_last_error().decode()}
        try:
            nv, nf, nm, dg = (_i64() for _ in range(4))
            self.L.rref_obj_info(h, C.byref(nv), C.byref(nf), C.byref(nm), C.byref(dg))
            v = np.zeros(max(nv.value, 1) * 3)
            f = np.zeros(max(nf.value, 1) * 4, np.int32)
            a = np.zeros(max(nm.value, 1) * 8)
            self.L.rref_obj_get(h, v, f, a)
            return {"ok": True, "vertices": v[: 3 * nv.value].reshape(-1, 3), "faces": f[: 4 * nf.value].reshape(-1, 4),
                    "absorption": a[: 8 * nm.value].reshape(-1, 8), "degenerate": dg.value}
        finally:
            self.L.rref_obj_free(h)

    def factors(self, dist, energy, c):
        """factors(build_pulse_trains(images, c)) (metrics.cpp:168-180):
        (9, 6, 2) array — bands 0..7 then mid; edt_s, t30_s, spl_db, c80_db,
        d50_pct, ts_ms; (value, reliable)."""
        dist = _c(dist, np.float64)
        out = np.zeros(9 * 6 * 2)
        if self.L.rref_factors(len(dist), dist, _c(energy, np.float64).reshape(-1), c, out):
            self._err()
        return out.reshape(9, 6, 2)

    def lattice(self, dims, walls_alpha, src, recv, max_distance, radius, air4):
        n = _i64()
        h = self.L.rref_lattice(_c(dims, np.float64), _c(walls_alpha, np.float64).reshape(-1),
                                _c(src, np.float64), _c(recv, np.float64), max_distance, radius,
                                _c(air4, np.float64), C.byref(n))
        if not h:
            self._err()
        n = n.value
        pos, dist, order, energy = np.empty((n, 3)), np.empty(n), np.empty(n, np.int32), np.empty((n, 8))
        self.L.rref_lattice_get(h, pos.reshape(-1), dist, order, energy.reshape(-1))
        hits = np.empty((n, 6), np.int32)
        self.L.rref_lattice_hits(h, hits.reshape(-1))
        self.L.rref_lattice_free(h)
        self.last_lattice_hits = hits
        return pos, dist, order, energy

    def compare(self, opos, oenergy, oorder, tpos, tenergy, pos_tol, tol_db):
        """The reference's compare (shoebox.cpp:126-182) -> dict of arrays."""
        opos, oen = _c(opos, np.float64).reshape(-1), _c(oenergy, np.float64).reshape(-1)
        tpos, ten = _c(tpos, np.float64).reshape(-1), _c(tenergy, np.float64).reshape(-1)
        oorder = _c(oorder, np.int32)
        counts, mx, rms = np.zeros(4, np.int64), C.c_double(), np.empty(8)
        h = self.L.rref_compare(len(oorder), opos, oen, oorder, len(tpos) // 3, tpos, ten, pos_tol, tol_db, counts,
                                C.byref(mx), rms)
        if not h:
            self._err()
        g, nm, nuo, nut = (int(x) for x in counts)
        r = dict(oracle_index=np.empty(g, np.int32), position_error=np.empty(g), order=np.empty(g, np.int32),
                 energy_delta_db=np.empty((g, 8)), member_off=np.empty(g + 1, np.int64),
                 members=np.empty(max(nm, 1), np.int32), unmatched_oracle=np.empty(max(nuo, 1), np.int32),
                 unmatched_traced=np.empty(max(nut, 1), np.int32))
        self.L.rref_compare_get(h, r["oracle_index"], r["position_error"], r["order"],
                                r["energy_delta_db"].reshape(-1), r["member_off"], r["members"],
                                r["unmatched_oracle"], r["unmatched_traced"])
        self.L.rref_compare_free(h)
        r["members"], r["unmatched_oracle"], r["unmatched_traced"] = (
            r["members"][:nm], r["unmatched_oracle"][:nuo], r["unmatched_traced"][:nut])
        r["max_position_error"], r["rms_energy_error_db"] = mx.value, rms
        return r

    def mesh_gen(self, kind: str, dims=(1.0, 1.0, 1.0), level=0):
        k = {"box": 0, "icosphere": 1, "tetra": 2}[kind]
        nv, nf = _i64(), _i64()
        h = self.L.rref_mesh_gen(k, _c(dims, np.float64), level, C.byref(nv), C.byref(nf))
        if not h:
            self._err()
        v, f = np.empty((nv.value, 3)), np.empty((nf.value, 4), np.int32)
        self.L.rref_mesh_get(h, v.reshape(-1), f.reshape(-1))
        self.L.rref_mesh_free(h)
        return v, f

    def hardware_threads(self):
        return self.L.rref_hardware_threads()


class RefScene:
    def __init__(self, ref: Ref, h, mesh: Mesh):
        self.r, self.h, self.mesh = ref, h, mesh

    def __del__(self):
        if getattr(self, "h", None):
            self.r.L.rref_scene_destroy(self.h)
            self.h = None

    def tree(self) -> Tree:
        root, depth = _i32(), _i32()
        n = self.r.L.rref_tree_size(self.h, C.byref(root), C.byref(depth))
        t = Tree(np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32),
                 np.empty((n, 3)), np.empty((n, 3)), root.value, depth.value)
        self.r.L.rref_tree_nodes(self.h, t.left, t.right, t.face, t.lo.reshape(-1), t.hi.reshape(-1))
        return t

    def nearest_hit(self, o, d, brute=False):
        o = _c(o, np.float64).reshape(-1, 3)
        d = _c(d, np.float64).reshape(-1, 3)
        n = len(o)
        face, delta, point = np.empty(n, np.int32), np.empty(n), np.empty((n, 3))
        if self.r.L.rref_nearest_hit(self.h, o.reshape(-1), d.reshape(-1), n, int(brute), face, delta,
                                     point.reshape(-1)):
            self.r._err()
        return face, delta, point

    def trace(self, src, ray_count, recv_center, radius, max_iterations=1000, max_range=0.0, threads=1,
              first=0, stride=0, count=0):
        h = self.r.L.rref_trace(self.h, _c(src, np.float64), ray_count, _c(recv_center, np.float64), radius,
                                max_iterations, max_range, threads, first, stride, count)
        if not h:
            self.r._err()
        try:
            it, tr = _i32(), _i32()
            esc, oor, nc, th, rb = (_i64() for _ in range(5))
            mr = C.c_double()
            self.r.L.rref_trace_info(h, C.byref(it), C.byref(tr), C.byref(esc), C.byref(oor), C.byref(mr),
                                     C.byref(nc), C.byref(th), C.byref(rb))
            n = nc.value
            cap = Captures(np.zeros(n, np.int32), np.empty(n, np.int32), np.empty((n, 3)), np.empty((n, 3)),
                           np.empty(n), np.empty((n, 8)), np.empty(n + 1, np.int64),
                           np.empty(max(th.value, 1), np.int32))
            self.r.L.rref_trace_captures(h, cap.ray, cap.point.reshape(-1), cap.dir.reshape(-1), cap.path,
                                         cap.mult.reshape(-1), cap.hist_off, cap.hist)
            cap.hist = cap.hist[:th.value]
            st = TraceStats(it.value, bool(tr.value), esc.value, oor.value, mr.value,
                            rb.value if stride > 0 else -1)
            return cap, st
        finally:
            self.r.L.rref_trace_free(h)

    def image_sources(self, cap: Captures, total_rays, air4, recv, tol_scale=1e-6, merge_coplanar=False):
        n = len(cap)
        h = self.r.L.rref_image_sources(self.h, n, _c(cap.ray, np.int32), _c(cap.point, np.float64).reshape(-1),
                                        _c(cap.dir, np.float64).reshape(-1), _c(cap.path, np.float64),
                                        _c(cap.mult, np.float64).reshape(-1), _c(cap.hist_off, np.int64),
                                        _c(cap.hist if len(cap.hist) else np.zeros(1), np.int32), total_rays,
                                        _c(air4, np.float64), _c(recv, np.float64), tol_scale,
                                        int(merge_coplanar))
        if not h:
            self.r._err()
        try:
            return _fetch_images(self.r.L.rref_images_info, self.r.L.rref_images_get, h)
        finally:
            self.r.L.rref_images_free(h)
