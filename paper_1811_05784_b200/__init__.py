"""roomray_b200 — B200-native specular ray / image-source engine.

Drop-in for the hot path of the roomray reference (arXiv 1811.05784):
median-split tree build, closest-hit traversal, reflection/absorption
bookkeeping, receiver capture, image sources and 8-band IR synthesis, as
hand-written sm_100a CUDA behind a C ABI (include/roomray_b200.h).
"""
from .roomray import (  # noqa: F401
    AccelTree, AirModel, Captures, Context, Receiver, RoomImpulseResponse, SourceConfig, TraceConfig,
    TraceResult, TriangleMesh, air_beta_bands, build_tree, design_band_filter, nearest_hit, nearest_hit_brute,
    reference_length, synthesize, trace, trace_device,
)
