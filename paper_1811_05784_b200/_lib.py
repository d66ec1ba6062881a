"""ctypes binding of libroomray_b200.so (the C ABI in include/roomray_b200.h).

The library is built in-tree by ``make -C paper_1811_05784_b200/csrc`` (see
``__graft_entry__.build``).  There is no fallback: if the shared object is
missing or no B200 is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# RR_LIB_PATH selects another build of the same ABI, e.g. the checked one
# (libroomray_b200_checked.so: device-side bounds checks, tests/test_gpu_checked.py)
LIB_PATH = os.environ.get("RR_LIB_PATH") or os.path.join(HERE, "libroomray_b200.so")

RR_OK, RR_INVALID_ARGUMENT, RR_RUNTIME, RR_CUDA, RR_NCCL = range(5)
RR_TRACE_NO_SMEM_CACHE = 1
RR_TRACE_KEEP_UNSORTED = 2
RR_TRACE_F32_LEAVES = 4
RR_TRACE_WIDE = 8
RR_TRACE_COUNT = 16
RR_TRACE_TREE8 = 32
RR_TRACE_TREE2 = 64

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double


class TreeNode(C.Structure):
    _fields_ = [("lo", _d * 3), ("hi", _d * 3), ("left", _i32), ("right", _i32), ("face_index", _i32),
                ("pad", _i32)]


class Source(C.Structure):
    _fields_ = [("position", _d * 3), ("ray_count", _i64)]


class Receiver(C.Structure):
    _fields_ = [("center", _d * 3), ("radius", _d)]


class TraceConfig(C.Structure):
    _fields_ = [("max_iterations", _i32), ("speed_of_sound", _d), ("max_range", _d), ("first", _i64),
                ("stride", _i64), ("count", _i64), ("block", _i64), ("flags", _i32),
                ("directions", _vp)]


class TraceStats(C.Structure):
    _fields_ = [("iterations", _i32), ("truncated", _i32), ("escaped", _i64), ("out_of_range", _i64),
                ("max_range", _d), ("n_captures", _i64), ("total_history", _i64), ("ray_bounces", _i64),
                ("n_rays", _i64), ("node_visits", _i64), ("leaf_tests", _i64), ("tree_width", _i32),
                ("node_bytes", _i32)]


class Air(C.Structure):
    _fields_ = [("enabled", _i32), ("temperature_c", _d), ("relative_humidity", _d), ("pressure_kpa", _d)]


class Metric(C.Structure):
    _fields_ = [("value", _d), ("reliable", _i32)]


class Factors(C.Structure):
    _fields_ = [("edt_s", Metric), ("t30_s", Metric), ("spl_db", Metric), ("c80_db", Metric), ("d50_pct", Metric),
                ("ts_ms", Metric)]


class ClusterOptions(C.Structure):
    _fields_ = [("tol_scale", _d), ("merge_coplanar", _i32)]


# (name, restype, argtypes) for every symbol of include/roomray_b200.h
SIGNATURES = [
    ("rr_last_error", C.c_char_p, []),
    ("rr_version", C.c_char_p, []),
    ("rr_ctx_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("rr_ctx_destroy", C.c_int, [_vp]),
    ("rr_ctx_stream", _vp, [_vp]),
    ("rr_ctx_launches", _i64, [_vp]),
    ("rr_host_alloc", C.c_int, [_i64, C.POINTER(_vp)]),
    ("rr_host_free", C.c_int, [_vp]),
    ("rr_scene_create", C.c_int, [_vp, _vp, _i64, _vp, _i64, _vp, _i32, _i32, C.POINTER(_vp)]),
    ("rr_scene_destroy", C.c_int, [_vp]),
    ("rr_scene_tree_info", C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i32)]),
    ("rr_scene_tree", C.c_int, [_vp, _vp]),
    ("rr_scene_normals", C.c_int, [_vp, _f64p]),
    ("rr_scene_build_ms", _d, [_vp]),
    ("rr_nearest_hit_batch", C.c_int, [_vp, _f64p, _f64p, _i64, _i32, _i32p, _f64p, _f64p]),
    ("rr_trace", C.c_int, [_vp, C.POINTER(Source), C.POINTER(Receiver), _i32, C.POINTER(TraceConfig),
                           C.POINTER(_vp)]),
    ("rr_trace_stats_get", C.c_int, [_vp, C.POINTER(TraceStats)]),
    ("rr_trace_captures", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("rr_captures_import", C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(Receiver), _i32,
                                     C.POINTER(_vp)]),
    ("rr_step", C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, C.POINTER(Receiver),
                          C.POINTER(TraceConfig), _i32, C.POINTER(_vp)]),
    ("rr_trace_kernel_ms", _d, [_vp]),
    ("rr_trace_destroy", C.c_int, [_vp]),
    ("rr_build_image_sources", C.c_int, [_vp, _i32, _i64, C.POINTER(Air), C.POINTER(ClusterOptions),
                                         C.POINTER(_vp)]),
    ("rr_images_info", C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    ("rr_images_get", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("rr_images_get_async", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("rr_images_destroy", C.c_int, [_vp]),
    ("rr_images_device", C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_i64)]),
    ("rr_air_beta_bands", C.c_int, [C.POINTER(Air), _f64p]),
    ("rr_band_schroeder", C.c_int, [_vp, _vp, _vp, _vp]),
    ("rr_air_alpha_db_per_m", C.c_int, [C.POINTER(Air), _d, C.POINTER(_d)]),
    ("rr_air_validate", C.c_int, [C.POINTER(Air)]),
    ("rr_fibonacci_directions", C.c_int, [_vp, _i64, _i64, _i64, _i64, _vp]),
    ("rr_shoebox_images", C.c_int, [_vp, _f64p, _f64p, _f64p, _f64p, _d, _d, C.POINTER(Air), C.POINTER(_vp)]),
    ("rr_lattice_info", C.c_int, [_vp, C.POINTER(_i64)]),
    ("rr_lattice_get", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    ("rr_lattice_destroy", C.c_int, [_vp]),
    ("rr_shoebox_compare", C.c_int, [_vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _d, _d, C.POINTER(_vp)]),
    ("rr_lattice_compare_images", C.c_int, [_vp, _vp, _d, _d, C.POINTER(_vp)]),
    ("rr_match_info", C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
                                C.POINTER(_d), _f64p]),
    ("rr_match_get", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("rr_match_destroy", C.c_int, [_vp]),
    ("rr_synthesize", C.c_int, [_vp, _i64, _f64p, _f64p, _d, _d, _i32, _i64, _vp, _vp]),
    ("rr_ir_bin_device", C.c_int, [_vp, _i64, _vp, _vp, _d, _d, _i64, _vp]),
    ("rr_ir_filter_device", C.c_int, [_vp, _vp, _d, _i32, _i64, _vp, _vp]),
    ("rr_synthesize_trains", C.c_int, [_vp, _i64p, _vp, _vp, _d, _i32, _i64, _vp, _vp]),
    ("rr_ir_reference_length", C.c_int, [_i64, _f64p, _d, _d, _i32, C.POINTER(_i64)]),
    ("rr_band_filter", C.c_int, [_i32, _d, _i32, _f64p]),
    ("rr_l2_read_gbs", C.c_int, [_vp, _i64, _i32, C.POINTER(_d)]),
    ("rr_band_factors", C.c_int, [_vp, _i64p, _vp, _vp, _vp]),
    ("rr_factors_from_images", C.c_int, [_vp, _i64, _vp, _vp, _d, _vp]),
    ("rr_images_factors", C.c_int, [_vp, _d, _vp]),
    ("rr_images_pulse_trains", C.c_int, [_vp, _d, _vp, _vp, _vp]),
    ("rr_pulse_trains", C.c_int, [_vp, _i64, _vp, _vp, _d, _vp, _vp, _vp]),
    ("rr_images_synthesize", C.c_int, [_vp, _d, _d, _i32, C.POINTER(_i64), _vp, _vp]),
    ("rr_comm_unique_id", C.c_int, [_vp]),
    ("rr_comm_init", C.c_int, [_vp, _vp, _i32, _i32, C.POINTER(_vp)]),
    ("rr_comm_info", C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    ("rr_hub_create", C.c_int, [_i32, C.POINTER(_vp)]),
    ("rr_hub_destroy", C.c_int, [_vp]),
    ("rr_comm_init_loopback", C.c_int, [_vp, _vp, _i32, C.POINTER(_vp)]),
    ("rr_comm_destroy", C.c_int, [_vp]),
    ("rr_pipeline_sharded", C.c_int, [_vp, _vp, C.POINTER(Source), C.POINTER(Receiver), _i32,
                                      C.POINTER(TraceConfig), C.POINTER(Air), C.POINTER(ClusterOptions), _d, _i64,
                                      _i32, _i32, C.POINTER(_vp)]),
    ("rr_sharded_info", C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64), _vp]),
    ("rr_sharded_take_images", C.c_int, [_vp, _i32, C.POINTER(_vp)]),
    ("rr_sharded_ir", C.c_int, [_vp, _i32, _vp, _vp]),
    ("rr_sharded_destroy", C.c_int, [_vp]),
]
RR_NCCL_ID_BYTES = 128

_LIB = None


def load(path: str = LIB_PATH):
    """Load (once) and bind the library; raises if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"libroomray_b200.so not built ({path}); run __graft_entry__.build()")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


class RoomrayError(RuntimeError):
    """RR_RUNTIME / RR_CUDA / RR_NCCL failures."""


def check(status: int) -> None:
    if status == RR_OK:
        return
    msg = _LIB.rr_last_error().decode()
    if status == RR_INVALID_ARGUMENT:
        raise ValueError(msg)  # the reference's std::invalid_argument
    raise RoomrayError(f"[status {status}] {msg}")


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data
