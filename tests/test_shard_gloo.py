"""Multi-rank exchange (paper_1811_05784_b200/shard.py) on CPU with gloo,
world size 2: each rank traces a strided shard of the lattice with the
oracle (standing in for its GPU), the captures are exchanged by order class,
each owner builds its image sources, the lists are gathered to rank 0 and
the pulse histograms summed.  The result must equal the single-process
oracle run on the whole lattice bit for bit (images) and to rounding (IR)."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1811_05784_b200 import scenes, shard  # noqa: E402

AIR = np.array([1.0, 20.0, 50.0, 101.325])
N_RAYS = 3000
MAX_IT = 12


def _scene():
    s = scenes.config1()
    return s


def _to_set(cap) -> shard.CaptureSet:
    t = torch.from_numpy
    return shard.CaptureSet(t(cap.ray.astype(np.int64)), t(cap.point.copy()), t(cap.dir.copy()), t(cap.path.copy()),
                            t(cap.mult.copy()), t(cap.hist_off.copy()), t(cap.hist[: cap.hist_off[-1]].copy()))


def _to_oracle(c: shard.CaptureSet):
    import oracle
    n = len(c)
    return oracle.Captures(np.zeros(n, np.int32), c.ray.numpy().astype(np.int32), c.point.numpy(), c.dir.numpy(),
                           c.path.numpy(), c.mult.numpy(), c.hist_off.numpy(), c.hist.numpy().astype(np.int32))


def _images_to_set(im) -> shard.ImageSet:
    t = torch.from_numpy
    return shard.ImageSet(t(im.pos), t(im.dist), t(im.energy), t(im.mult), t(im.ray_count), t(im.order),
                          t(im.has_proj), t(im.proj), t(im.path_off), t(im.path[: im.path_off[-1]].astype(np.int32)))


def _synth(port, im, fs, taps, length):
    out = np.zeros(length)
    if len(im):
        got = np.zeros(length)
        port_len = port.synthesize(im.dist, im.energy, 343.0, fs, taps)
        got[: min(length, len(port_len))] = port_len[:length]
        out += got
    return out


def _worker(rank, world, port_no, merge, q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = _scene()
        port = oracle.Port()
        sc = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
        (rc, rr) = s.receivers[0]
        cap, _ = sc.trace(s.source, N_RAYS, [rc], [rr], MAX_IT, s.max_range, 1, rank, world, 0)
        mine = _to_set(cap)
        owner = shard.order_owners(mine, MAX_IT)
        got = shard.exchange_captures(mine, owner)
        # every capture this rank received belongs to an order class it owns
        assert all(owner[o] == rank for o in got.order.tolist())
        im = sc.image_sources(_to_oracle(got), N_RAYS, AIR, np.array(rc), 1e-6, merge)
        local = _images_to_set(im)
        merged = shard.gather_images(local)
        L = 4096
        hist = torch.from_numpy(_synth(port, im, 44100.0, 1023, L))
        shard.reduce_histogram(hist)
        if rank == 0:
            q.put(("ok", {k: getattr(merged, k).numpy() for k in merged.__dataclass_fields__}, hist.numpy()))
    except Exception as e:  # surface the failure to the parent
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("merge", [False, True])
def test_two_rank_exchange_matches_single_process(port, merge):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, pn, merge, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, images, hist = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", images
    assert all(p.exitcode == 0 for p in procs)

    s = _scene()
    sc = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    (rc, rr) = s.receivers[0]
    cap, _ = sc.trace(s.source, N_RAYS, [rc], [rr], MAX_IT, s.max_range)
    ref = sc.image_sources(cap, N_RAYS, AIR, np.array(rc), 1e-6, merge)
    assert len(ref) > 20
    assert np.array_equal(images["order"], ref.order)
    assert np.array_equal(images["ray_count"], ref.ray_count)
    assert np.array_equal(images["position"], ref.pos)
    assert np.array_equal(images["distance"], ref.dist)
    assert np.array_equal(images["band_energy"], ref.energy)
    assert np.array_equal(images["band_multiplier"], ref.mult)
    assert np.array_equal(images["has_projection"], ref.has_proj)
    assert np.array_equal(images["projection"], ref.proj)
    assert np.array_equal(images["path_off"], ref.path_off)
    assert np.array_equal(images["path"], ref.path[: ref.path_off[-1]])
    full = _synth(port, ref, 44100.0, 1023, 4096)
    np.testing.assert_allclose(hist, full, rtol=1e-9, atol=1e-12 * np.abs(full).max())


def test_assign_orders_is_balanced_and_deterministic():
    counts = [0, 50, 40, 30, 30, 20, 10, 5, 0, 1]
    a = shard.assign_orders(counts, 3)
    assert a == shard.assign_orders(counts, 3)
    load = [sum(c for c, o in zip(counts, a) if o == r) for r in range(3)]
    assert max(load) - min(load) <= max(counts)
    assert shard.assign_orders(counts, 1) == [0] * len(counts)


def test_sort_reference_order_and_csr_gather():
    off = torch.tensor([0, 2, 2, 5, 6])
    hist = torch.tensor([1, 2, 3, 4, 5, 6], dtype=torch.int32)
    c = shard.CaptureSet(torch.tensor([7, 3, 3, 1]), torch.zeros(4, 3, dtype=torch.float64),
                         torch.zeros(4, 3, dtype=torch.float64), torch.arange(4, dtype=torch.float64),
                         torch.zeros(4, 8, dtype=torch.float64), off, hist)
    s = shard.sort_reference_order(c)
    assert s.ray.tolist() == [1, 3, 3, 7]
    assert s.order.tolist() == [1, 0, 3, 2]
    assert s.hist.tolist() == [6, 3, 4, 5, 1, 2]
    assert s.path.tolist() == [3.0, 1.0, 2.0, 0.0]
    sel = shard.select(c, torch.tensor([False, True, True, False]))
    assert sel.hist_off.tolist() == [0, 0, 3] and sel.hist.tolist() == [3, 4, 5]
