"""Host API mirroring the reference's C++ interface for the hot path.

Same names, argument meaning and error behaviour as namespace ``roomray``
(/root/reference/proj/include/roomray): ``build_tree`` (accel_tree.hpp:38),
``nearest_hit`` / ``nearest_hit_brute`` (accel_tree.hpp:50-55), ``trace``
(tracer.hpp:50-52), ``build_image_sources`` (image_sources.hpp:58-61),
``air_beta_bands`` (air_absorption.hpp:30), ``build_pulse_trains`` +
``synthesize`` (rir.hpp:33-45), ``design_band_filter`` (rir.hpp:38).
``std::invalid_argument`` surfaces as ``ValueError``.  Everything runs through
the C ABI of libroomray_b200.so on the GPU; there is no CPU path.
Vectorised: queries take (n, 3) arrays where the reference takes one ray.
"""
from __future__ import annotations

import atexit
import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, ptr

# Device handles are not released during interpreter shutdown (the CUDA
# runtime may already be torn down); the process exit reclaims them.
_SHUTDOWN = []
atexit.register(lambda: _SHUTDOWN.append(True))

NUM_BANDS = 8
BAND_CENTERS_HZ = (62.5, 125.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0, 8000.0)
BAND_FILTER_TAPS = 1023
SELF_HIT_EPSILON = 1e-6


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


class Context:
    """One CUDA device + stream (rr_ctx)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.rr_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    @property
    def stream(self) -> int:
        return self.lib.rr_ctx_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return self.lib.rr_ctx_launches(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.rr_ctx_destroy(self.h)
            self.h = None


@dataclass
class TriangleMesh:
    """TriangleMesh (geometry.hpp:60-77) as arrays: vertices (nv,3) f64,
    faces (nf,4) i32 [a, b, c, material_id], absorption (nmat,8) f64."""

    vertices: np.ndarray
    faces: np.ndarray
    absorption: np.ndarray

    def __post_init__(self):
        self.vertices = _f64(self.vertices).reshape(-1, 3)
        self.faces = np.ascontiguousarray(self.faces, dtype=np.int32).reshape(-1, 4)
        self.absorption = _f64(self.absorption).reshape(-1, NUM_BANDS)

    def face_count(self) -> int:
        return len(self.faces)

    def bounds(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)


class AccelTree:
    """Device scene (rr_scene): faces, a device SAH traversal tree, and the
    reference-layout median-split tree, built on first use of nodes()."""

    def __init__(self, mesh: TriangleMesh, ctx: Context | None = None, validate: bool = True):
        self.ctx = ctx or Context.default()
        self.lib = self.ctx.lib
        self.mesh = mesh
        h = C.c_void_p()
        check(self.lib.rr_scene_create(self.ctx.h, ptr(mesh.vertices), len(mesh.vertices), ptr(mesh.faces),
                                       len(mesh.faces), ptr(mesh.absorption), len(mesh.absorption), int(validate),
                                       C.byref(h)))
        self.h = h
        n, root, depth = C.c_int64(), C.c_int32(), C.c_int32()
        check(self.lib.rr_scene_tree_info(self.h, C.byref(n), C.byref(root), C.byref(depth)))
        self._n, self.root, self._depth = n.value, root.value, depth.value

    def __del__(self):
        if getattr(self, "h", None) and not _SHUTDOWN:
            self.lib.rr_scene_destroy(self.h)
            self.h = None

    def node_count(self) -> int:
        return self._n

    def depth(self) -> int:
        return self._depth

    def nodes(self) -> dict:
        """Reference-layout nodes (TreeNode accel_tree.hpp:15-22)."""
        arr = (_lib.TreeNode * self._n)()
        check(self.lib.rr_scene_tree(self.h, C.cast(arr, C.c_void_p)))
        raw = np.frombuffer(arr, dtype=np.dtype([("lo", "f8", 3), ("hi", "f8", 3), ("left", "i4"),
                                                 ("right", "i4"), ("face", "i4"), ("pad", "i4")]))
        return {k: np.array(raw[k]) for k in ("lo", "hi", "left", "right", "face")}

    def leaf_count(self) -> int:
        return int((self.nodes()["face"] >= 0).sum())

    def normals(self) -> np.ndarray:
        out = np.empty((len(self.mesh.faces), 3))
        check(self.lib.rr_scene_normals(self.h, out.reshape(-1)))
        return out

    @property
    def build_ms(self) -> float:
        return self.lib.rr_scene_build_ms(self.h)


def build_tree(mesh: TriangleMesh, ctx: Context | None = None, validate: bool = True) -> AccelTree:
    """build_tree (accel_tree.hpp:38): the device scene and its trees."""
    return AccelTree(mesh, ctx, validate)


def _hits(tree: AccelTree, origins, dirs, brute: bool):
    o = _f64(origins).reshape(-1, 3)
    d = _f64(dirs).reshape(-1, 3)
    if o.shape != d.shape:
        raise ValueError("origins and dirs must have the same shape")
    n = len(o)
    face = np.empty(n, np.int32)
    delta = np.empty(n)
    point = np.empty((n, 3))
    check(tree.lib.rr_nearest_hit_batch(tree.h, o.reshape(-1), d.reshape(-1), n, int(brute), face, delta,
                                        point.reshape(-1)))
    return face, delta, point


def nearest_hit(tree: AccelTree, origins, dirs):
    """nearest_hit (accel_tree.hpp:50-51) for n rays -> (face, delta, point);
    face = -1 where the reference returns std::nullopt."""
    return _hits(tree, origins, dirs, False)


def nearest_hit_brute(tree: AccelTree, origins, dirs):
    """nearest_hit_brute (accel_tree.hpp:54-55)."""
    return _hits(tree, origins, dirs, True)


@dataclass
class SourceConfig:
    position: tuple = (0.0, 0.0, 0.0)
    ray_count: int = 1


@dataclass
class Receiver:
    center: tuple = (0.0, 0.0, 0.0)
    radius: float = 0.1


@dataclass
class TraceConfig:
    """TraceConfig (tracer.hpp:13-20).  thread_count is accepted for API
    compatibility and ignored (the GPU grid replaces it)."""

    max_iterations: int = 1000
    speed_of_sound: float = 343.0
    max_range: float = 0.0
    thread_count: int = 1


@dataclass
class Captures:
    """Capture records (tracer_types.hpp:27-34) as sorted arrays."""

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

    def select(self, mask) -> "Captures":
        idx = np.nonzero(mask)[0]
        lens = self.hist_off[idx + 1] - self.hist_off[idx]
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        hist = np.concatenate([self.history(i) for i in idx]) if len(idx) else np.zeros(0, np.int32)
        return Captures(self.recv[idx], self.ray[idx], self.point[idx], self.dir[idx], self.path[idx],
                        self.mult[idx], off, hist.astype(np.int32))


@dataclass
class TraceResult:
    """TraceResult (tracer.hpp:22-29) + ray_bounces and kernel time."""

    captures: Captures
    iterations: int
    truncated: bool
    escaped: int
    out_of_range: int
    max_range: float
    ray_bounces: int
    n_rays: int
    kernel_ms: float


class DeviceTrace:
    """A trace whose captures are still on the device (rr_trace_result)."""

    def __init__(self, tree: AccelTree, h):
        self.tree, self.h, self.lib = tree, h, tree.lib
        st = _lib.TraceStats()
        check(self.lib.rr_trace_stats_get(self.h, C.byref(st)))
        self.stats = st

    def __del__(self):
        if getattr(self, "h", None) and not _SHUTDOWN:
            self.lib.rr_trace_destroy(self.h)
            self.h = None

    @property
    def kernel_ms(self) -> float:
        return self.lib.rr_trace_kernel_ms(self.h)

    def captures(self) -> Captures:
        n = self.stats.n_captures
        th = self.stats.total_history
        c = Captures(np.empty(n, np.int32), np.empty(n, np.int32), np.empty((n, 3)), np.empty((n, 3)),
                     np.empty(n), np.empty((n, NUM_BANDS)), np.empty(n + 1, np.int64),
                     np.empty(max(th, 1), np.int32))
        check(self.lib.rr_trace_captures(self.h, ptr(c.recv), ptr(c.ray), ptr(c.point), ptr(c.dir), ptr(c.path),
                                         ptr(c.mult), ptr(c.hist_off), ptr(c.hist)))
        c.hist = c.hist[:th]
        return c

    def result(self) -> TraceResult:
        s = self.stats
        return TraceResult(self.captures(), s.iterations, bool(s.truncated), s.escaped, s.out_of_range,
                           s.max_range, s.ray_bounces, s.n_rays, self.kernel_ms)


def trace_device(tree: AccelTree, source: SourceConfig, receivers, config: TraceConfig = TraceConfig(), *,
                 first: int = 0, stride: int = 0, count: int = 0, block: int = 0, flags: int = 0,
                 directions: np.ndarray | None = None) -> DeviceTrace:
    recs = receivers if isinstance(receivers, (list, tuple)) else [receivers]
    src = _lib.Source((C.c_double * 3)(*map(float, source.position)), int(source.ray_count))
    rarr = (_lib.Receiver * len(recs))(*[_lib.Receiver((C.c_double * 3)(*map(float, r.center)), float(r.radius))
                                         for r in recs])
    dirs = None if directions is None else _f64(directions).reshape(-1, 3)
    cfg = _lib.TraceConfig(int(config.max_iterations), float(config.speed_of_sound), float(config.max_range),
                           int(first), int(stride), int(count), int(block), int(flags), ptr(dirs))
    h = C.c_void_p()
    check(tree.lib.rr_trace(tree.h, C.byref(src), rarr, len(recs), C.byref(cfg), C.byref(h)))
    return DeviceTrace(tree, h)


def trace(tree: AccelTree, source: SourceConfig, receivers, config: TraceConfig = TraceConfig(),
          **subset) -> TraceResult:
    """trace (tracer.hpp:50-52).  ``receivers`` may be one Receiver or a list
    (each capture records its receiver index).  ``subset`` keywords
    (first/stride/count or block-cyclic first=rank, stride=world, block=B)
    select part of the N-ray lattice; ``directions`` (count x 3) replaces the
    device-evaluated lattice with caller rays (the Ray span of step(),
    tracer.hpp:43)."""
    return trace_device(tree, source, receivers, config, **subset).result()


@dataclass
class AirModel:
    """AirModel (air_absorption.hpp:10-23)."""

    temperature_c: float = 20.0
    relative_humidity: float = 50.0
    pressure_kpa: float = 101.325
    enabled: bool = True

    @staticmethod
    def off() -> "AirModel":
        return AirModel(enabled=False)

    def c(self):
        return _lib.Air(int(self.enabled), self.temperature_c, self.relative_humidity, self.pressure_kpa)


def air_alpha_db_per_m(air: AirModel, frequency: float) -> float:
    """air_alpha_db_per_m (air_absorption.cpp:21-53), dB/m."""
    lib = _lib.load()
    out = C.c_double()
    a = air.c()
    check(lib.rr_air_alpha_db_per_m(C.byref(a), float(frequency), C.byref(out)))
    return out.value


def air_validate(air: AirModel) -> None:
    """AirModel::validate (air_absorption.cpp:8-19): ValueError out of range."""
    lib = _lib.load()
    a = air.c()
    check(lib.rr_air_validate(C.byref(a)))


def fibonacci_directions(n: int, first: int = 0, stride: int = 1, count: int | None = None,
                         ctx: Context | None = None) -> np.ndarray:
    """fibonacci_directions (emission.cpp:17-29) evaluated on the device the
    way the tracer emits its rays (glibc's sincos restated bit for bit,
    rr_sincos.cuh)."""
    ctx = ctx or Context.default()
    if count is None:
        count = max(0, (n - first + stride - 1) // stride) if n >= 1 else 0
    out = np.empty((count, 3))
    check(ctx.lib.rr_fibonacci_directions(ctx.h, int(n), int(first), int(stride), int(count), ptr(out)))
    return out


def air_beta_bands(air: AirModel) -> np.ndarray:
    lib = _lib.load()
    out = np.empty(NUM_BANDS)
    a = air.c()
    check(lib.rr_air_beta_bands(C.byref(a), out))
    return out


def design_band_filter(band: int, sample_rate: float, taps: int = BAND_FILTER_TAPS) -> np.ndarray:
    """design_band_filter (rir.cpp:32-58), tap count parameterised."""
    lib = _lib.load()
    out = np.empty(taps)
    check(lib.rr_band_filter(band, sample_rate, taps, out))
    return out


def reference_length(distance, speed_of_sound: float, sample_rate: float, taps: int = BAND_FILTER_TAPS) -> int:
    lib = _lib.load()
    d = _f64(distance).reshape(-1)
    out = C.c_int64()
    check(lib.rr_ir_reference_length(len(d), d, speed_of_sound, sample_rate, taps, C.byref(out)))
    return out.value


@dataclass
class RoomImpulseResponse:
    """RoomImpulseResponse (rir.hpp:26-30) + the per-band responses."""

    sample_rate: float
    samples: np.ndarray
    band_ir: np.ndarray


def synthesize(distance, band_energy, speed_of_sound: float, sample_rate: float, taps: int = BAND_FILTER_TAPS,
               length: int | None = None, ctx: Context | None = None) -> RoomImpulseResponse:
    """build_pulse_trains + synthesize (rir.hpp:33-45) from image distances
    and band energies.  ``length`` None = the reference's length
    (rir.cpp:78-80)."""
    ctx = ctx or Context.default()
    d = _f64(distance).reshape(-1)
    e = _f64(band_energy).reshape(-1, NUM_BANDS)
    if len(d) != len(e):
        raise ValueError("distance and band_energy disagree in length")
    if length is None:
        length = reference_length(d, speed_of_sound, sample_rate, taps)
        if length == 0:
            return RoomImpulseResponse(sample_rate, np.zeros(0), np.zeros((NUM_BANDS, 0)))
    band = np.empty((NUM_BANDS, length))
    bb = np.empty(length)
    check(ctx.lib.rr_synthesize(ctx.h, len(d), d, e.reshape(-1), speed_of_sound, sample_rate, taps, length,
                                ptr(band), ptr(bb)))
    return RoomImpulseResponse(sample_rate, bb, band)


@dataclass
class ClusterOptions:
    """ClusterOptions (image_sources.hpp:25-31)."""

    tol_scale: float = 1e-6
    merge_coplanar: bool = False


@dataclass
class ImageSources:
    """ImageSource list (image_sources.hpp:14-23) as arrays, sorted by
    (order, distance, face path)."""

    position: np.ndarray
    distance: np.ndarray
    band_energy: np.ndarray
    band_multiplier: np.ndarray
    ray_count: np.ndarray
    order: np.ndarray
    has_projection: np.ndarray
    projection: np.ndarray
    path_off: np.ndarray
    path: np.ndarray

    def __len__(self):
        return len(self.distance)

    def face_path(self, i):
        return self.path[self.path_off[i]:self.path_off[i + 1]]


class DeviceImages:
    """Image sources resident on the device (rr_images)."""

    def __init__(self, lib, h):
        self.lib, self.h = lib, h
        n, tp = C.c_int64(), C.c_int64()
        check(lib.rr_images_info(h, C.byref(n), C.byref(tp)))
        self.n, self.total_path = n.value, tp.value

    def __del__(self):
        if getattr(self, "h", None) and not _SHUTDOWN:
            self.lib.rr_images_destroy(self.h)
            self.h = None

    def fetch(self, alloc=np.empty) -> ImageSources:
        """Copy to host arrays made by alloc(shape, dtype) (numpy's by default;
        pass a pinned-memory allocator for full-bandwidth copies)."""
        n = self.n
        f8, i4 = np.float64, np.int32
        im = ImageSources(alloc((n, 3), f8), alloc((n,), f8), alloc((n, NUM_BANDS), f8), alloc((n, NUM_BANDS), f8),
                          alloc((n,), i4), alloc((n,), i4), alloc((n,), i4), alloc((n, 3), f8),
                          alloc((n + 1,), np.int64), alloc((max(self.total_path, 1),), i4))
        check(self.lib.rr_images_get(self.h, ptr(im.position), ptr(im.distance), ptr(im.band_energy),
                                     ptr(im.band_multiplier), ptr(im.ray_count), ptr(im.order),
                                     ptr(im.has_projection), ptr(im.projection), ptr(im.path_off), ptr(im.path)))
        im.path = im.path[:self.total_path]
        return im

    def device_arrays(self):
        """(dist device ptr, energy device ptr, n) for rr_ir_bin_device."""
        d, e, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(self.lib.rr_images_device(self.h, C.byref(d), C.byref(e), C.byref(n)))
        return d.value, e.value, n.value


def import_captures(tree: AccelTree, ray, point, direction, path, histories, receiver: Receiver,
                    mult=None) -> DeviceTrace:
    """rr_captures_import: caller-held Capture records (tracer_types.hpp:27-34)
    as a device trace for build_image_sources (image_sources.hpp:58-61).
    ``histories`` is a list of face-index sequences; ``mult`` None rebuilds
    the multipliers from the histories (the product of 1 - alpha)."""
    n = len(ray)
    r = np.ascontiguousarray(ray, np.int32).reshape(-1)
    lens = np.array([len(h) for h in histories], np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    hist = np.ascontiguousarray(np.concatenate([np.asarray(h, np.int32) for h in histories]) if lens.sum()
                                else np.zeros(1, np.int32), np.int32)
    pt, di, pa = _f64(point).reshape(n, 3), _f64(direction).reshape(n, 3), _f64(path).reshape(n)
    m = None if mult is None else _f64(mult).reshape(n, NUM_BANDS)
    rec = _lib.Receiver((C.c_double * 3)(*map(float, receiver.center)), float(receiver.radius))
    h = C.c_void_p()
    check(tree.lib.rr_captures_import(tree.h, n, None, ptr(r), ptr(pt), ptr(di), ptr(pa), ptr(m), ptr(off),
                                      ptr(hist), C.byref(rec), 1, C.byref(h)))
    return DeviceTrace(tree, h)


def build_image_sources_device(trace_res: DeviceTrace, total_rays: int, air: AirModel = AirModel(),
                               options: ClusterOptions = ClusterOptions(), receiver: int = 0) -> DeviceImages:
    a = air.c()
    o = _lib.ClusterOptions(float(options.tol_scale), int(options.merge_coplanar))
    h = C.c_void_p()
    check(trace_res.lib.rr_build_image_sources(trace_res.h, int(receiver), int(total_rays), C.byref(a), C.byref(o),
                                               C.byref(h)))
    return DeviceImages(trace_res.lib, h)


def build_image_sources(trace_res: DeviceTrace, total_rays: int, air: AirModel = AirModel(),
                        options: ClusterOptions = ClusterOptions(), receiver: int = 0) -> ImageSources:
    """build_image_sources (image_sources.hpp:58-61) for one receiver of a
    device trace (captures never leave the GPU)."""
    return build_image_sources_device(trace_res, total_rays, air, options, receiver).fetch()


# ------------------------------------------------------------------ shoebox lattice (shoebox.hpp)
@dataclass
class OracleImages:
    """OracleImageSource list (shoebox.hpp:25-31), sorted by (distance, cell)."""

    position: np.ndarray
    distance: np.ndarray
    order: np.ndarray
    wall_hits: np.ndarray
    band_energy: np.ndarray

    def __len__(self):
        return len(self.distance)


class Lattice:
    """enumerate_images result resident on the device (rr_lattice)."""

    def __init__(self, lib, h):
        self.lib, self.h = lib, h
        n = C.c_int64()
        check(lib.rr_lattice_info(h, C.byref(n)))
        self.n = n.value

    def __len__(self):
        return self.n

    def __del__(self):
        if getattr(self, "h", None) and not _SHUTDOWN:
            self.lib.rr_lattice_destroy(self.h)
            self.h = None

    def fetch(self) -> OracleImages:
        n = self.n
        o = OracleImages(np.empty((n, 3)), np.empty(n), np.empty(n, np.int32), np.empty((n, 6), np.int32),
                         np.empty((n, NUM_BANDS)))
        check(self.lib.rr_lattice_get(self.h, ptr(o.position), ptr(o.distance), ptr(o.order), ptr(o.wall_hits),
                                      ptr(o.band_energy)))
        return o


def enumerate_images(dimensions, walls_alpha, source, receiver, max_distance: float, receiver_radius: float,
                     air: AirModel = AirModel(), ctx: Context | None = None) -> Lattice:
    """enumerate_images (shoebox.hpp:38-43) on the device: every mirror image of
    `source` in the box [0, L]^3 within max_distance of `receiver`; walls
    x0, x1, y0, y1, z0, z1 with 8-band absorption walls_alpha (6, 8)."""
    ctx = ctx or Context.default()
    a = air.c()
    h = C.c_void_p()
    check(ctx.lib.rr_shoebox_images(ctx.h, _f64(dimensions, (3,)), _f64(walls_alpha, (6 * NUM_BANDS,)),
                                    _f64(source, (3,)), _f64(receiver, (3,)), float(max_distance),
                                    float(receiver_radius), C.byref(a), C.byref(h)))
    return Lattice(ctx.lib, h)


@dataclass
class MatchReport:
    """MatchReport (shoebox.hpp:56-66); matched images in oracle order."""

    oracle_index: np.ndarray
    position_error: np.ndarray
    order: np.ndarray
    energy_delta_db: np.ndarray
    member_off: np.ndarray
    members: np.ndarray
    unmatched_oracle: np.ndarray
    unmatched_traced: np.ndarray
    max_position_error: float
    rms_energy_error_db: np.ndarray
    pos_tol: float
    energy_tol_db: float

    def traced_indices(self, i):
        return self.members[self.member_off[i]:self.member_off[i + 1]]

    def energy_within(self, tol_db: float, max_order: int) -> bool:
        """MatchReport::energy_within (shoebox.cpp:118-124)."""
        sel = self.order <= max_order
        return not bool((np.abs(self.energy_delta_db[sel]) > tol_db).any())


def compare(oracle, traced, pos_tol: float, energy_tol_db: float, ctx: Context | None = None) -> MatchReport:
    """compare (shoebox.hpp:67-70) on the device.  `oracle` is a Lattice or
    OracleImages; `traced` a DeviceImages, ImageSources or (position, energy)."""
    h = C.c_void_p()
    if isinstance(oracle, Lattice) and isinstance(traced, DeviceImages):
        lib = oracle.lib
        check(lib.rr_lattice_compare_images(oracle.h, traced.h, float(pos_tol), float(energy_tol_db), C.byref(h)))
    else:
        ctx = ctx or Context.default()
        lib = ctx.lib
        if isinstance(oracle, Lattice):
            oracle = oracle.fetch()
        if isinstance(traced, DeviceImages):
            traced = traced.fetch()
        if isinstance(traced, tuple):
            tp, te = traced
        else:
            tp, te = traced.position, traced.band_energy
        op, oe = _f64(oracle.position).reshape(-1, 3), _f64(oracle.band_energy).reshape(-1, NUM_BANDS)
        oo = np.ascontiguousarray(oracle.order, np.int32)
        tp, te = _f64(tp).reshape(-1, 3), _f64(te).reshape(-1, NUM_BANDS)
        check(lib.rr_shoebox_compare(ctx.h, len(op), ptr(op), ptr(oe), ptr(oo), len(tp), ptr(tp), ptr(te),
                                     float(pos_tol), float(energy_tol_db), C.byref(h)))
    try:
        g, nm, nuo, nut = (C.c_int64() for _ in range(4))
        mx = C.c_double()
        rms = np.empty(NUM_BANDS)
        check(lib.rr_match_info(h, C.byref(g), C.byref(nm), C.byref(nuo), C.byref(nut), C.byref(mx), rms))
        n = g.value
        r = MatchReport(np.empty(n, np.int32), np.empty(n), np.empty(n, np.int32), np.empty((n, NUM_BANDS)),
                        np.empty(n + 1, np.int64), np.empty(nm.value, np.int32), np.empty(nuo.value, np.int32),
                        np.empty(nut.value, np.int32), mx.value, rms, float(pos_tol), float(energy_tol_db))
        check(lib.rr_match_get(h, ptr(r.oracle_index), ptr(r.position_error), ptr(r.order), ptr(r.energy_delta_db),
                               ptr(r.member_off), ptr(r.members), ptr(r.unmatched_oracle), ptr(r.unmatched_traced)))
        return r
    finally:
        lib.rr_match_destroy(h)


FACTOR_NAMES = ("edt_s", "t30_s", "spl_db", "c80_db", "d50_pct", "ts_ms")


def _factors_out(arr) -> dict:
    """9 rr_factors -> {"bands": [8 x {name: (value, reliable)}], "mid": {...}}."""
    conv = [{k: (getattr(f, k).value, bool(getattr(f, k).reliable)) for k in FACTOR_NAMES} for f in arr]
    return {"bands": conv[:NUM_BANDS], "mid": conv[NUM_BANDS]}


def factors(distance, band_energy, speed_of_sound: float = 343.0, ctx: Context | None = None) -> dict:
    """factors(build_pulse_trains(images, c)) (metrics.hpp:56-60, rir.hpp:33)
    on the device: per band EDT, T30, SPL, C80, D50, Ts and the 500 Hz -
    1 kHz "mid" average, each as (value, reliable)."""
    ctx = ctx or Context.default()
    d = _f64(distance).reshape(-1)
    e = _f64(band_energy).reshape(-1, NUM_BANDS)
    out = (_lib.Factors * 9)()
    check(ctx.lib.rr_factors_from_images(ctx.h, len(d), ptr(d), ptr(e), float(speed_of_sound),
                                         C.cast(out, C.c_void_p)))
    return _factors_out(out)


def factors_of_images(images: "DeviceImages", speed_of_sound: float = 343.0) -> dict:
    """factors() of a device image set without leaving the GPU."""
    out = (_lib.Factors * 9)()
    check(images.lib.rr_images_factors(images.h, float(speed_of_sound), C.cast(out, C.c_void_p)))
    return _factors_out(out)


@dataclass
class Rays:
    """A span of Ray (tracer_types.hpp:11-18) as SoA arrays for step():
    origin/dir (n,3), mult (n,8), path (n,), alive (n,) int32, hist
    (n, hist_cap) int32 face history with n_hist (n,) entries used.  numpy
    arrays (host) or CUDA tensors (device, updated in place)."""

    origin: object
    dir: object
    mult: object
    path: object
    alive: object
    hist: object
    n_hist: object

    @staticmethod
    def emit(source: SourceConfig, hist_cap: int, directions=None) -> "Rays":
        """emit (emission.cpp:31-43): rays at the source with multiplier 1;
        directions default to the Fibonacci lattice (host, the oracle-free
        numpy restatement of emission.cpp:17-29)."""
        n = int(source.ray_count)
        if directions is None:
            k = np.arange(n, dtype=np.float64)
            z = 1.0 - (2.0 * k + 1.0) / n
            rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
            phi = (2.0 * math.pi * (1.0 - 1.0 / ((1.0 + math.sqrt(5.0)) / 2.0))) * k
            directions = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], 1)
        return Rays(np.tile(np.asarray(source.position, np.float64), (n, 1)), _f64(directions).reshape(n, 3).copy(),
                    np.ones((n, NUM_BANDS)), np.zeros(n), np.ones(n, np.int32), np.zeros((n, hist_cap), np.int32),
                    np.zeros(n, np.int32))


def _vptr(a):
    return C.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)


def step(tree: AccelTree, rays: Rays, receiver: Receiver, config: TraceConfig = TraceConfig(),
         brute: bool = False) -> DeviceTrace:
    """step (tracer.hpp:43-45): one iteration over `rays` in place; returns
    this iteration's captures (DeviceTrace.captures(), .kernel_ms)."""
    n = len(rays.path)
    hist_cap = rays.hist.shape[1]
    rec = _lib.Receiver((C.c_double * 3)(*map(float, receiver.center)), float(receiver.radius))
    cfg = _lib.TraceConfig(int(config.max_iterations), float(config.speed_of_sound), float(config.max_range), 0, 0, 0,
                           0, 0, None)
    h = C.c_void_p()
    check(tree.lib.rr_step(tree.h, n, _vptr(rays.origin), _vptr(rays.dir), _vptr(rays.mult), _vptr(rays.path),
                           _vptr(rays.alive), _vptr(rays.hist), _vptr(rays.n_hist), int(hist_cap), C.byref(rec),
                           C.byref(cfg), int(brute), C.byref(h)))
    return DeviceTrace(tree, h)


# ------------------------------------------------------------------ multi-GPU through the C ABI
class Comm:
    """An NCCL communicator bound to a Context (rr_comm): one per rank.  The
    unique id (rr_comm_unique_id, 128 bytes) comes from rank 0 and reaches
    the others out of band (e.g. torch.distributed.broadcast_object_list)."""

    @staticmethod
    def unique_id() -> bytes:
        lib = _lib.load()
        buf = (C.c_uint8 * _lib.RR_NCCL_ID_BYTES)()
        check(lib.rr_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        self.ctx, self.lib = ctx, ctx.lib
        buf = (C.c_uint8 * _lib.RR_NCCL_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        check(self.lib.rr_comm_init(ctx.h, buf, int(nranks), int(rank), C.byref(h)))
        self.h, self.rank, self.nranks = h, rank, nranks

    @classmethod
    def loopback(cls, ctx: Context, hub: "Hub", rank: int) -> "Comm":
        """Rank `rank` of an in-process loopback hub (testing the multi-rank
        exchange on one GPU: one thread and one Context per rank)."""
        c = cls.__new__(cls)
        c.ctx, c.lib = ctx, ctx.lib
        h = C.c_void_p()
        check(c.lib.rr_comm_init_loopback(ctx.h, hub.h, int(rank), C.byref(h)))
        c.h, c.rank, c.nranks, c.hub = h, rank, hub.nranks, hub
        return c

    def __del__(self):
        if getattr(self, "h", None) and not _SHUTDOWN:
            self.lib.rr_comm_destroy(self.h)
            self.h = None


class Hub:
    """rr_hub: the rendezvous of in-process loopback ranks (see Comm.loopback)."""

    def __init__(self, nranks: int):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.rr_hub_create(int(nranks), C.byref(h)))
        self.h, self.nranks = h, nranks

    def __del__(self):
        if getattr(self, "h", None) and not _SHUTDOWN:
            self.lib.rr_hub_destroy(self.h)
            self.h = None


@dataclass
class PipelineResult:
    """Per receiver: images[r] (rank 0: every rank's image sources in the
    reference order; other ranks: empty), band_ir[r] (8, L), broadband[r]
    (L,); this rank's ray_bounces / n_rays, image sources built here, and
    stage times (ms) trace / exchange / images / ir / gather."""

    images: list
    band_ir: list
    broadband: list
    ray_bounces: int
    n_rays: int
    local_images: int
    stage_ms: dict


def pipeline_sharded(tree: AccelTree, source: SourceConfig, receivers, config: TraceConfig = TraceConfig(), *,
                     comm: Comm | None = None, air: AirModel = AirModel(), options: ClusterOptions = ClusterOptions(),
                     sample_rate: float = 48000.0, length: int | None = None, taps: int = 1023, block: int = 4096,
                     device_images: bool = False, alloc=np.empty) -> PipelineResult:
    """run_trace_pipeline's trace -> image sources -> IRs (pipeline.cpp:163-175)
    on the device, over the ranks of `comm` (rr_pipeline_sharded); comm=None
    is the single-GPU pipeline.  Captures never leave the GPU.  Host outputs
    go to arrays made by alloc(shape, dtype) (e.g. pinned memory)."""
    recs = receivers if isinstance(receivers, (list, tuple)) else [receivers]
    src = _lib.Source((C.c_double * 3)(*map(float, source.position)), int(source.ray_count))
    rarr = (_lib.Receiver * len(recs))(*[_lib.Receiver((C.c_double * 3)(*map(float, r.center)), float(r.radius))
                                         for r in recs])
    cfg = _lib.TraceConfig(int(config.max_iterations), float(config.speed_of_sound), float(config.max_range), 0, 0, 0,
                           0, 0, None)
    a = air.c()
    o = _lib.ClusterOptions(float(options.tol_scale), int(options.merge_coplanar))
    if length is None:
        length = int(round(2.0 * sample_rate))
    h = C.c_void_p()
    lib = tree.lib
    check(lib.rr_pipeline_sharded(tree.h, comm.h if comm is not None else None, C.byref(src), rarr, len(recs),
                                  C.byref(cfg), C.byref(a), C.byref(o), float(sample_rate), int(length), int(taps),
                                  int(block), C.byref(h)))
    try:
        rb, nr, li = C.c_int64(), C.c_int64(), C.c_int64()
        ms = (C.c_float * 5)()
        check(lib.rr_sharded_info(h, C.byref(rb), C.byref(nr), C.byref(li), ms))
        images, bands, bbs = [], [], []
        for r in range(len(recs)):
            ih = C.c_void_p()
            check(lib.rr_sharded_take_images(h, r, C.byref(ih)))
            di = DeviceImages(lib, ih)
            images.append(di if device_images else di.fetch(alloc))
            band = alloc((NUM_BANDS, length), np.float64)
            bb = alloc((length,), np.float64)
            check(lib.rr_sharded_ir(h, r, band.ctypes.data, bb.ctypes.data))
            bands.append(band)
            bbs.append(bb)
        names = ("trace", "exchange", "images", "ir", "gather")
        return PipelineResult(images, bands, bbs, rb.value, nr.value, li.value,
                              {k: float(v) for k, v in zip(names, ms)})
    finally:
        lib.rr_sharded_destroy(h)
