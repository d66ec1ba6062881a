"""rr_pipeline_sharded: the multi-GPU pipeline behind the C ABI
(run_trace_pipeline's trace -> image sources -> IRs, pipeline.cpp:163-175).

Only one GPU is available to the tests, so the exchange path runs on a
one-rank NCCL communicator: order-class histogram all-reduce, LPT ownership,
destination sort, packing and the grouped send/recv all-to-all (self copies
on one rank), capture import in the reference order, the global fixed-point
scale of the pulse histograms (max / sum all-reduce), the exact integer
all-reduce, and the image gather to rank 0.  Its results must equal the
plain device pipeline (comm=None) and the step-by-step API bit for bit, and
the oracle's images / impulse responses (BASELINE tolerance for the IR band
energies, 1e-4 relative).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh, scenes
from paper_1811_05784_b200 import roomray as rr

pytestmark = pytest.mark.gpu

AIR = (1.0, 20.0, 50.0, 101.325)


@pytest.fixture(scope="module")
def comm1(ctx):
    return rr.Comm(ctx, rr.Comm.unique_id(), 1, 0)


def _images_equal(a, b):
    assert len(a.distance) == len(b.distance)
    for k in ("position", "distance", "band_energy", "band_multiplier", "ray_count", "order", "has_projection",
              "projection", "path_off", "path"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)


def _run(ctx, s, comm, merge, n=None, fs=None, length=None):
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    recvs = [Receiver(c, r) for c, r in s.receivers]
    fs = fs or s.sample_rate
    length = length or int(round(s.ir_seconds * fs))
    return tree, rr.pipeline_sharded(tree, SourceConfig(s.source, n or s.ray_count), recvs,
                                     TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range), comm=comm,
                                     options=rr.ClusterOptions(1e-6, merge), sample_rate=fs, length=length)


@pytest.mark.parametrize("cfg,merge", [("c1", True), ("c2", False), ("c3", True)])
def test_exchange_path_equals_device_pipeline(ctx, comm1, cfg, merge):
    s = scenes.CONFIGS[cfg]()
    _, plain = _run(ctx, s, None, merge)
    _, xch = _run(ctx, s, comm1, merge)
    assert plain.ray_bounces == xch.ray_bounces and plain.n_rays == xch.n_rays == s.ray_count
    assert plain.local_images == xch.local_images > 0
    for r in range(len(s.receivers)):
        _images_equal(plain.images[r], xch.images[r])
        np.testing.assert_array_equal(plain.band_ir[r], xch.band_ir[r])
        np.testing.assert_array_equal(plain.broadband[r], xch.broadband[r])
    assert set(xch.stage_ms) == {"trace", "exchange", "images", "ir", "gather"}


def test_device_pipeline_equals_step_by_step_api(ctx):
    s = scenes.config1()
    tree, res = _run(ctx, s, None, True)
    dt = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), [Receiver(*s.receivers[0])],
                         TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range))
    im = rr.build_image_sources(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True))
    _images_equal(res.images[0], im)
    L = int(round(s.ir_seconds * s.sample_rate))
    syn = rr.synthesize(im.distance, im.band_energy, 343.0, s.sample_rate, taps=1023, length=L, ctx=ctx)
    np.testing.assert_array_equal(res.band_ir[0], syn.band_ir)
    np.testing.assert_array_equal(res.broadband[0], syn.samples)


def test_pipeline_against_oracle(ctx, comm1, port):
    s = scenes.config1()
    _, res = _run(ctx, s, comm1, True)
    rc, rad = s.receivers[0]
    ps = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    oc, _ = ps.trace(s.source, s.ray_count, [rc], [rad], s.max_iterations, s.max_range)
    oi = ps.image_sources(oc, s.ray_count, AIR, rc, 1e-6, True)
    g = res.images[0]
    assert len(g.distance) == len(oi.dist) > 100
    np.testing.assert_array_equal(g.position, oi.pos)
    np.testing.assert_array_equal(g.distance, oi.dist)
    np.testing.assert_array_equal(g.path, oi.path)
    np.testing.assert_allclose(g.band_energy, oi.energy, rtol=1e-12, atol=0)
    L = res.band_ir[0].shape[1]
    for b in range(8):
        want = port.synthesize(oi.dist, oi.energy, 343.0, s.sample_rate, 1023, 1 << b)[:L]
        got = res.band_ir[0][b][:len(want)]
        eg, ew = float((got ** 2).sum()), float((want ** 2).sum())
        assert abs(eg - ew) <= 1e-4 * ew, (b, eg, ew)  # north_star: band IR energy 1e-4 relative


def test_comm_errors(ctx):
    with pytest.raises(ValueError):
        rr.Comm(ctx, rr.Comm.unique_id(), 2, 5)  # rank out of range
