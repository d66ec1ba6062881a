"""GPU parity on the BASELINE.json configurations beyond C1/C2:

* C3 (436 000-triangle open amphitheatre, 5 receivers): device tree equal to
  build_tree; a strided lattice subset traced bit for bit against the oracle
  (escapes, captures of all 5 receivers, face paths, multipliers).
* C5 (2 000 000-triangle scatterer room): device tree equal to build_tree;
  a strided subset of the 8 * 10^6-ray lattice, 100 reflections, bit for bit.
* C4 (IR synthesis only, 2 * 10^6 image sources, 2 048 taps): per-band
  responses against the oracle's synthesize on a subset (BASELINE tolerance:
  band energies 1e-4 relative), and at full size against an FFT convolution
  of a numpy-binned pulse histogram, plus linearity (the property that lets
  per-GPU histograms be summed).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh, trace
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    return scenes.config3()


@pytest.fixture(scope="module")
def c5():
    return scenes.config5()


def _tree_equal(gpu, ot):
    g = gpu.nodes()
    assert gpu.node_count() == len(ot.left) and gpu.root == ot.root and gpu.depth() == ot.depth
    for k, o in (("left", ot.left), ("right", ot.right), ("face", ot.face), ("lo", ot.lo), ("hi", ot.hi)):
        np.testing.assert_array_equal(g[k], o)


def _subset_trace(ctx, port, s, stride, first=1):
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    cnt = (s.ray_count - first + stride - 1) // stride
    dirs = port.fibonacci(s.ray_count, first, stride, cnt)
    recvs = [Receiver(c, r) for c, r in s.receivers]
    res = trace(tree, SourceConfig(s.source, s.ray_count), recvs,
                TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range), directions=dirs, first=first,
                stride=stride)
    sc = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    oc, ost = sc.trace(s.source, s.ray_count, [c for c, _ in s.receivers], [r for _, r in s.receivers],
                       s.max_iterations, s.max_range, 8, first, stride, 0)
    return tree, sc, res, oc, ost


def _captures_equal(g, o):
    assert len(g) == len(o), (len(g), len(o))
    for k in ("ray", "recv", "hist_off", "path", "point", "dir", "mult"):
        np.testing.assert_array_equal(getattr(g, k), getattr(o, k), err_msg=k)
    np.testing.assert_array_equal(g.hist, o.hist[: o.hist_off[-1]])


def test_c3_tree_and_trace_subset(ctx, port, c3):
    tree, sc, res, oc, ost = _subset_trace(ctx, port, c3, stride=50)
    _tree_equal(tree, sc.tree())
    assert res.escaped == ost.escaped > 0  # open air: rays leave the scene
    assert res.out_of_range == ost.out_of_range and res.ray_bounces == ost.ray_bounces
    assert (res.iterations, res.truncated) == (ost.iterations, ost.truncated)
    _captures_equal(res.captures, oc)
    assert len(np.unique(oc.recv)) == 5


def test_c5_tree_and_trace_subset(ctx, port, c5):
    tree, sc, res, oc, ost = _subset_trace(ctx, port, c5, stride=4000)
    _tree_equal(tree, sc.tree())
    assert res.ray_bounces == ost.ray_bounces == 100 * res.n_rays  # closed room, cap reached
    assert res.truncated and ost.truncated
    _captures_equal(res.captures, oc)
    assert len(oc) > 100


# ---------------------------------------------------------------- C4
@pytest.fixture(scope="module")
def c4():
    return scenes.config4()


def _gpu_synth(ctx, dist, energy, fs, taps, length):
    out = rr.synthesize(dist, energy, 343.0, fs, taps=taps, length=length, ctx=ctx)
    return out.band_ir, out.samples


def test_c4_subset_per_band_vs_oracle(ctx, port, c4):
    n = 20_000
    d, e = c4["distance"][:n], c4["energy"][:n]
    fs, taps = c4["sample_rate"], c4["taps"]
    length = rr.reference_length(d, 343.0, fs, taps)
    band, bb = _gpu_synth(ctx, d, e, fs, taps, length)
    for b in range(8):
        want = port.synthesize(d, e, 343.0, fs, taps, 1 << b)
        assert len(want) == length
        eg, ew = float((band[b] ** 2).sum()), float((want ** 2).sum())
        assert abs(eg - ew) <= 1e-4 * ew, (b, eg, ew)  # north_star: band IR energy 1e-4 relative
        np.testing.assert_allclose(band[b], want, rtol=0, atol=1e-9 * np.abs(want).max())
    np.testing.assert_allclose(bb, band.sum(0), rtol=0, atol=1e-12 * np.abs(bb).max())


def _np_hist(d, e, c, fs, length):
    centre = np.floor(d / c * fs + 0.5).astype(np.int64)  # lround for t >= 0
    ok = centre < length
    h = np.zeros((8, length))
    a = np.sqrt(e)
    for b in range(8):
        h[b] = np.bincount(centre[ok], weights=a[ok, b], minlength=length)[:length]
    return h


def test_c4_full_size_vs_fft_convolution(ctx, port, c4):
    d, e = c4["distance"], c4["energy"]
    fs, taps = c4["sample_rate"], c4["taps"]
    length = int(round(c4["seconds"] * fs))
    band, bb = _gpu_synth(ctx, d, e, fs, taps, length)
    h = _np_hist(d, e, 343.0, fs, length + taps)
    delay = (taps - 1) // 2
    for b in range(8):
        k = port.band_filter(b, fs, taps)
        m = len(h[b]) + taps - 1
        nfft = 1 << (m - 1).bit_length()
        full = np.fft.irfft(np.fft.rfft(h[b], nfft) * np.fft.rfft(k, nfft), nfft)[:m]
        want = full[delay: delay + length]  # out[j] = sum_n h[j + delay - n] k[n]
        np.testing.assert_allclose(band[b], want, rtol=0, atol=1e-9 * np.abs(want).max())
    # linearity: two halves synthesized separately sum to the whole
    half = len(d) // 2
    b1, _ = _gpu_synth(ctx, d[:half], e[:half], fs, taps, length)
    b2, _ = _gpu_synth(ctx, d[half:], e[half:], fs, taps, length)
    np.testing.assert_allclose(b1 + b2, band, rtol=0, atol=1e-12 * np.abs(band).max())


def test_c4_device_histogram_checksum(ctx, c4):
    """sum over samples of the band histogram == sum of sqrt(E) (all events
    land inside the 3 s window), per band."""
    d, e = c4["distance"], c4["energy"]
    n = len(d)
    L = int(round(c4["seconds"] * c4["sample_rate"]))
    dd = torch.from_numpy(d).cuda()
    de = torch.from_numpy(e.reshape(-1)).cuda()
    hist = torch.empty(8 * L, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    rr._lib.check(ctx.lib.rr_ir_bin_device(ctx.h, n, C.c_void_p(dd.data_ptr()), C.c_void_p(de.data_ptr()), 343.0,
                                           c4["sample_rate"], L, C.c_void_p(hist.data_ptr())))
    torch.cuda.synchronize()
    got = hist.view(8, L).sum(1).cpu().numpy()
    want = np.sqrt(e).sum(0)
    np.testing.assert_allclose(got, want, rtol=1e-12)
