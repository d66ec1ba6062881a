"""rr_pipeline_sharded: the multi-GPU pipeline behind the C ABI
(run_trace_pipeline's trace -> image sources -> IRs, pipeline.cpp:163-175).

Only one GPU is available to the tests, so the exchange runs (1) on a
one-rank NCCL communicator -- the NCCL calls themselves -- and (2) on 2-4
in-process loopback ranks (rr_hub: one thread, context and replicated scene
per rank on the same GPU; the collectives rendezvous on the hub and copy on
the device), which exercises the multi-rank logic proper: block-cyclic
shards, the summed order histogram, LPT ownership, the cross-rank
all-to-all of capture records, capture import in the reference order, the
global fixed-point scale of the pulse histograms and their exact integer
sum, and the image gather to rank 0.  Results must equal the plain device
pipeline (comm=None) and the step-by-step API bit for bit, and the oracle's
images / impulse responses (BASELINE tolerance for the IR band energies,
1e-4 relative).
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


# ---------------------------------------------------------------- several ranks on one GPU
def _run_ranks(s, world, merge, block):
    """world loopback ranks (one thread + one context + one replicated scene
    each) through rr_pipeline_sharded; returns every rank's result."""
    import threading

    from paper_1811_05784_b200 import Context
    hub = rr.Hub(world)
    ctxs = [Context(0) for _ in range(world)]
    trees = [AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), c) for c in ctxs]
    comms = [rr.Comm.loopback(c, hub, r) for r, c in enumerate(ctxs)]
    recvs = [Receiver(c, r) for c, r in s.receivers]
    L = int(round(s.ir_seconds * s.sample_rate))
    out, err = [None] * world, []

    def rank(r):
        try:
            out[r] = rr.pipeline_sharded(trees[r], SourceConfig(s.source, s.ray_count), recvs,
                                         TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                                         comm=comms[r], options=rr.ClusterOptions(1e-6, merge),
                                         sample_rate=s.sample_rate, length=L, block=block)
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    return out


@pytest.mark.parametrize("cfg,world,merge,block", [("c1", 2, True, 512), ("c1", 3, True, 4096),
                                                   ("c2", 2, False, 4096), ("c3", 4, True, 4096)])
def test_multi_rank_exchange_equals_one_gpu(ctx, cfg, world, merge, block):
    """The multi-rank path proper -- block-cyclic shards, summed order
    histograms, LPT ownership over several ranks, cross-rank all-to-all of the
    capture records, the global fixed-point IR scale and integer sum, the
    image gather -- on loopback ranks, against one GPU, bit for bit."""
    s = scenes.CONFIGS[cfg]()
    _, one = _run(ctx, s, None, merge)
    res = _run_ranks(s, world, merge, block)
    assert sum(r.n_rays for r in res) == s.ray_count
    assert sum(r.ray_bounces for r in res) == one.ray_bounces
    assert sum(r.local_images for r in res) == one.local_images
    assert sum(r.local_images > 0 for r in res) > 1  # the image work really was split
    if cfg == "c3":  # (receiver, order) units owned jointly: 5 receivers x ~4 orders over 4 ranks
        loads = [r.local_images for r in res]
        assert min(loads) > 0 and max(loads) <= 2 * sum(loads) / world, loads
    for rcv in range(len(s.receivers)):
        _images_equal(res[0].images[rcv], one.images[rcv])
        for r in range(world):
            np.testing.assert_array_equal(res[r].band_ir[rcv], one.band_ir[rcv])
            np.testing.assert_array_equal(res[r].broadband[rcv], one.broadband[rcv])
            if r:
                assert len(res[r].images[rcv].distance) == 0
