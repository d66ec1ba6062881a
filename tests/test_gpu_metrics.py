"""Perceptive factors (metrics.cpp:62-180) on the device vs the unmodified
reference (oracle/_ref): per band EDT, T30, SPL, C80, D50, Ts and the mid
average.  The device sums in parallel, the reference sequentially, so values
are compared to 1e-6 relative; reliability flags must match exactly."""
import numpy as np
import pytest

from paper_1811_05784_b200 import AccelTree, Receiver, SourceConfig, TraceConfig, TriangleMesh
from paper_1811_05784_b200 import roomray as rr
from paper_1811_05784_b200 import scenes

pytestmark = pytest.mark.gpu


def _compare(got: dict, want: np.ndarray, rtol=1e-6):
    rows = got["bands"] + [got["mid"]]
    for b, row in enumerate(rows):
        for k, name in enumerate(rr.FACTOR_NAMES):
            v, rel = row[name]
            wv, wr = want[b, k]
            assert rel == bool(wr), (b, name, row[name], want[b, k])
            assert abs(v - wv) <= rtol * max(abs(wv), 1e-3), (b, name, v, wv)


def test_factors_exponential_decay(ctx, ref):
    """Dense diffuse-like decay: every factor reliable, T30 close to the
    decay constant it was drawn from."""
    n = 200_000
    u = scenes.uniform(77, 2 * n).reshape(n, 2)
    d = 3.0 + 340.0 * u[:, 0]  # 0.009 .. 1 s
    tau = 0.05  # E ~ exp(-t / tau): -60 dB after 6 ln(10) tau = 0.69 s
    e = np.exp(-(d / 343.0) / tau)[:, None] * (0.5 + u[:, 1:2]) * np.linspace(1.0, 0.3, 8)[None, :]
    got = rr.factors(d, e, 343.0, ctx=ctx)
    want = ref.factors(d, e, 343.0)
    _compare(got, want)
    t30 = got["bands"][4]["t30_s"]
    assert t30[1] and abs(t30[0] - 60.0 * tau / (10.0 * np.log10(np.e))) < 0.05


def test_factors_traced_room(ctx, ref, port):
    s = scenes.config1()
    tree = AccelTree(TriangleMesh(s.vertices, s.faces, s.absorption), ctx)
    dt = rr.trace_device(tree, SourceConfig(s.source, s.ray_count), Receiver(*s.receivers[0]),
                         TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                         directions=port.fibonacci(s.ray_count))
    dimg = rr.build_image_sources_device(dt, s.ray_count, rr.AirModel(), rr.ClusterOptions(1e-6, True))
    im = dimg.fetch()
    assert len(im) > 50
    want = ref.factors(im.distance, im.band_energy, 343.0)
    _compare(rr.factors(im.distance, im.band_energy, 343.0, ctx=ctx), want)
    _compare(rr.factors_of_images(dimg, 343.0), want)


def test_factors_edge_cases(ctx, ref):
    # no events: every factor unreliable (metrics.cpp:124)
    got = rr.factors(np.zeros(0), np.zeros((0, 8)), 343.0, ctx=ctx)
    assert all(not v[1] for row in got["bands"] for v in row.values())
    # one silent band, the rest single early events (C80 clamps to +99 dB)
    d = np.array([5.0, 7.0, 9.0])
    e = np.ones((3, 8))
    e[:, 2] = 0.0
    got = rr.factors(d, e, 343.0, ctx=ctx)
    _compare(got, ref.factors(d, e, 343.0))
    assert not got["bands"][2]["spl_db"][1]
    assert got["bands"][0]["c80_db"] == (99.0, True)
    with pytest.raises(ValueError):
        rr.factors(d, e, 0.0, ctx=ctx)
