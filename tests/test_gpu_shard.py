"""GPU side of the multi-GPU exchange on one B200, without collectives:
block-cyclic shards are traced one after another, their captures are split
by order class exactly as shard.exchange_captures routes them, each owner's
part is imported (rr_captures_import) and turned into image sources on the
device, and the per-owner lists are merged like shard.gather_images.  The
result must equal the single-trace image list bit for bit, and the summed
per-owner pulse histograms must equal the single-trace histogram."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes, shard

pytestmark = pytest.mark.gpu

FIELDS = ("position", "distance", "band_energy", "band_multiplier", "ray_count", "order", "has_projection",
          "projection", "path_off", "path")


def _cat_sets(parts):
    off, n0, h0 = [torch.zeros(1, dtype=torch.int64, device="cuda")], 0, 0
    for p in parts:
        off.append(p.hist_off[1:] + h0)
        h0 += int(p.hist_off[-1])
    return shard.CaptureSet(torch.cat([p.ray for p in parts]), torch.cat([p.point for p in parts]),
                            torch.cat([p.dir for p in parts]), torch.cat([p.path for p in parts]),
                            torch.cat([p.mult for p in parts]), torch.cat(off), torch.cat([p.hist for p in parts]))


def _merge_images(parts):
    """shard.gather_images without the collective."""
    n = [len(p) for p in parts]
    off = [torch.zeros(1, dtype=torch.int64, device="cuda")]
    h0 = 0
    for p in parts:
        off.append(p.path_off[1:] + h0)
        h0 += int(p.path_off[-1])
    cat = shard.ImageSet(*[torch.cat([getattr(p, f) for p in parts]) for f in FIELDS[:8]], torch.cat(off),
                         torch.cat([p.path for p in parts]))
    perm = torch.sort(cat.order.to(torch.int64), stable=True).indices
    poff, path = shard._csr_gather(cat.path_off, cat.path, perm)
    return shard.ImageSet(*[getattr(cat, f)[perm] for f in FIELDS[:8]], poff, path)


@pytest.mark.parametrize("merge", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_images_equal_single_trace(ctx, merge, world):
    s = scenes.config1()
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    n_rays = 6000
    src = rr.SourceConfig(s.source, n_rays)
    recv = rr.Receiver(*s.receivers[0])
    cfg = rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    opts = rr.ClusterOptions(1e-6, merge)
    full = rr.trace_device(tree, src, recv, cfg)
    ref = shard.images_to_tensors(rr.build_image_sources_device(full, n_rays, rr.AirModel(), opts))
    assert len(ref) > 50
    # per-rank block-cyclic shards (block 256 so every rank gets several blocks)
    parts = [shard.device_captures(rr.trace_device(tree, src, recv, cfg, first=r, stride=world, block=256), 0)
             for r in range(world)]
    allc = _cat_sets(parts)
    assert len(allc) == full.stats.n_captures
    owner = shard.assign_orders(shard.order_counts(allc, cfg.max_iterations).cpu().tolist(), world)
    own = torch.tensor(owner, device="cuda")
    per_owner = []
    hist_sum = None
    L, taps = 8192, 1023
    for q in range(world):
        mine = shard.sort_reference_order(shard.select(allc, own[allc.order] == q))
        dt = shard.import_captures(tree, mine, recv)
        dimg = rr.build_image_sources_device(dt, n_rays, rr.AirModel(), opts)
        per_owner.append(shard.images_to_tensors(dimg))
        d_dist, d_en, n_img = dimg.device_arrays()
        h = torch.empty(8 * (L + taps), dtype=torch.float64, device="cuda")
        if n_img:
            tree.lib.rr_ir_bin_device(ctx.h, n_img, C.c_void_p(d_dist), C.c_void_p(d_en), 343.0, 44100.0, L + taps,
                                      C.c_void_p(h.data_ptr()))
        else:
            h.zero_()
        torch.cuda.synchronize()
        hist_sum = h if hist_sum is None else hist_sum + h
    got = _merge_images(per_owner)
    for f in FIELDS:
        a, b = getattr(got, f).cpu().numpy(), getattr(ref, f).cpu().numpy()
        assert np.array_equal(a, b), f
    full_img = rr.build_image_sources_device(full, n_rays, rr.AirModel(), opts)  # keep alive while binning
    d_dist, d_en, n_img = full_img.device_arrays()
    h_ref = torch.empty(8 * (L + taps), dtype=torch.float64, device="cuda")
    tree.lib.rr_ir_bin_device(ctx.h, n_img, C.c_void_p(d_dist), C.c_void_p(d_en), 343.0, 44100.0, L + taps,
                              C.c_void_p(h_ref.data_ptr()))
    torch.cuda.synchronize()
    h_ref = h_ref.cpu().numpy()
    # fixed-point binning: per-call quantum max_amp * n * 2^-62
    np.testing.assert_allclose(hist_sum.cpu().numpy(), h_ref, rtol=0, atol=1e-12 * np.abs(h_ref).max())
    assert np.abs(h_ref).max() > 0


def test_import_roundtrip_equals_trace(ctx):
    """device_captures -> rr_captures_import (mult rebuilt from history and
    given) reproduces the trace's own capture arrays."""
    s = scenes.config1()
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    dt = rr.trace_device(tree, rr.SourceConfig(s.source, 3000), rr.Receiver(*s.receivers[0]),
                         rr.TraceConfig(max_iterations=20, max_range=s.max_range))
    c = shard.device_captures(dt)
    perm = torch.randperm(len(c), device="cuda")
    off, hist = shard._csr_gather(c.hist_off, c.hist, perm)
    shuffled = shard.CaptureSet(c.ray[perm], c.point[perm], c.dir[perm], c.path[perm], c.mult[perm], off, hist)
    a = dt.captures()
    for mult in (True, False):
        sc = shuffled if mult else shard.CaptureSet(shuffled.ray, shuffled.point, shuffled.dir, shuffled.path,
                                                     None, shuffled.hist_off, shuffled.hist)
        if not mult:
            imp = _import_no_mult(tree, sc, rr.Receiver(*s.receivers[0]))
        else:
            imp = shard.import_captures(tree, sc, rr.Receiver(*s.receivers[0]))
        b = imp.captures()
        for f in ("ray", "point", "dir", "path", "mult", "hist_off", "hist"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (f, mult)


def _import_no_mult(tree, c, receiver):
    from paper_1811_05784_b200 import _lib
    rarr = (_lib.Receiver * 1)(_lib.Receiver((C.c_double * 3)(*map(float, receiver.center)), float(receiver.radius)))
    ts = [c.ray.to(torch.int32).contiguous(), c.point.contiguous(), c.dir.contiguous(), c.path.contiguous(),
          c.hist_off.contiguous(), c.hist.contiguous()]
    vp = [C.c_void_p(t.data_ptr()) for t in ts]
    h = C.c_void_p()
    torch.cuda.synchronize()
    _lib.check(tree.lib.rr_captures_import(tree.h, len(c), None, vp[0], vp[1], vp[2], vp[3], None, vp[4], vp[5],
                                           rarr, 1, C.byref(h)))
    return rr.DeviceTrace(tree, h)


def test_import_rejects_bad_records(ctx):
    s = scenes.config1()
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    c = shard.CaptureSet(torch.tensor([0], device="cuda"), torch.zeros((1, 3), dtype=torch.float64, device="cuda"),
                         torch.zeros((1, 3), dtype=torch.float64, device="cuda"),
                         torch.zeros(1, dtype=torch.float64, device="cuda"), None,
                         torch.tensor([0, 1], device="cuda"), torch.tensor([10 ** 6], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        _import_no_mult(tree, c, rr.Receiver(*s.receivers[0]))


def test_nccl_exchange_path_single_rank():
    """The collective path of run_sharded through NCCL (one rank, forced)."""
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "native", "nccl_single.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "exchange ok" in r.stdout


@pytest.mark.parametrize("cfg_name", ["c1", "c3"])
def test_host_fetch_equals_device_results(ctx, cfg_name):
    """run_sharded(host=True) (image list copied to pinned host memory on a
    side stream while the IR stage runs) returns exactly the device results,
    for one receiver (C1) and five (C3)."""
    s = scenes.CONFIGS[cfg_name]()
    tree = rr.AccelTree(rr.TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    src = rr.SourceConfig(s.source, 20000)
    recv = [rr.Receiver(*r) for r in s.receivers]
    cfg = rr.TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range)
    L = int(round(0.25 * s.sample_rate))
    kw = dict(air=rr.AirModel(), options=rr.ClusterOptions(1e-6, True), sample_rate=s.sample_rate, length=L)
    dev = shard.run_sharded(tree, src, recv, cfg, **kw)
    host = shard.run_sharded(tree, src, recv, cfg, host=True, **kw)
    torch.cuda.synchronize()
    assert len(host.images) == len(dev.images) == len(recv)
    for r in range(len(recv)):
        assert len(host.images[r]) == len(dev.images[r]) > 0
        for f in FIELDS:
            h, d = getattr(host.images[r], f), getattr(dev.images[r], f)
            assert not h.is_cuda and h.is_pinned()
            assert torch.equal(h, d.cpu()), (r, f)
        assert not host.band_ir[r].is_cuda and torch.equal(host.band_ir[r], dev.band_ir[r].cpu())
        assert torch.equal(host.broadband[r], dev.broadband[r].cpu())
