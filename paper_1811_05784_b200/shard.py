"""Multi-GPU sharding of the trace and the exchange step,
over torch.distributed: the Python mirror of the library's rr_pipeline_sharded
(csrc/rr_shard.cu), kept for the world-size-2 gloo tests on CPU
(tests/test_shard_gloo.py, the oracle as per-rank compute).  The product
path is rr_pipeline_sharded; this mirror assigns order classes per receiver
(the library assigns (receiver, order) units jointly) and sums fp64 pulse
histograms (the library sums 64-bit fixed-point ones, bit-exactly).

Rays shard (the reference already chunks them, tracer.cpp:82-105): every
rank holds the replicated mesh + tree and traces a block-cyclic shard of
the global Fibonacci lattice.  Nothing is exchanged while tracing.  The one
exchange step turns per-rank captures into one image-source list and one
set of band impulse responses:

1. ``order_owners``: ``all_reduce`` of the per-order capture histogram, then
   a deterministic longest-processing-time assignment of *order classes*
   (face-path lengths) to ranks.  The reference groups captures by exact face
   path (image_sources.cpp:87-90), splits within a group and merges coplanar
   images only between equal orders (image_sources.cpp:111-116), so an order
   class is closed under all of it; the greedy merge inside a class depends
   only on the path order within the class.  Hence owning whole classes is
   exact on any number of ranks.
2. ``exchange_captures``: ``all_to_all_single`` of fixed-width capture records
   (global ray, path length, point, direction, path, 8 band multipliers) and
   of the face histories to the owners; ``sort_reference_order`` restores the
   reference order (ray index, path length; tracer.cpp:143-147).
3. owners build their image sources (K5 on their GPU; energy uses the global
   N, image_sources.cpp:138);
4. ``reduce_histogram``: 8-band pulse histograms summed with ``all_reduce``
   (binning and FIR are linear), then one FIR pass;
5. ``gather_images``: image lists to rank 0, stably ordered by order class
   (inside a class the owner's order already is the reference's
   (order, distance, path) order, image_sources.cpp:163-168).

The collectives go through ``torch.distributed`` (NCCL over NVLink on the
GPUs; gloo in the CPU tests, where the oracle stands in for the per-rank
compute).  Tensors may live on any device the process group supports.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

NUM_BANDS = 8
# capture record: ray, order, point(3), dir(3), path, mult(8)
CAP_FIELDS = 2 + 3 + 3 + 1 + NUM_BANDS
# image record: pos(3), dist, energy(8), mult(8), ray_count, order, has_proj, proj(3), path_len
IMG_FIELDS = 3 + 1 + NUM_BANDS + NUM_BANDS + 1 + 1 + 1 + 3 + 1


@dataclass
class CaptureSet:
    """Captures of one receiver as tensors (Capture, tracer_types.hpp:27-34):
    ray (n,) int64 global lattice index, point/dir (n,3) f64, path (n,) f64,
    mult (n,8) f64, hist_off (n+1,) int64, hist (H,) int32."""

    ray: torch.Tensor
    point: torch.Tensor
    dir: torch.Tensor
    path: torch.Tensor
    mult: torch.Tensor
    hist_off: torch.Tensor
    hist: torch.Tensor

    def __len__(self):
        return int(self.ray.numel())

    @property
    def order(self) -> torch.Tensor:
        return self.hist_off[1:] - self.hist_off[:-1]

    @staticmethod
    def empty(device="cpu") -> "CaptureSet":
        f = dict(dtype=torch.float64, device=device)
        return CaptureSet(torch.zeros(0, dtype=torch.int64, device=device), torch.zeros((0, 3), **f),
                          torch.zeros((0, 3), **f), torch.zeros(0, **f), torch.zeros((0, NUM_BANDS), **f),
                          torch.zeros(1, dtype=torch.int64, device=device),
                          torch.zeros(0, dtype=torch.int32, device=device))


@dataclass
class ImageSet:
    """Image sources (ImageSource, image_sources.hpp:14-23) as tensors."""

    position: torch.Tensor
    distance: torch.Tensor
    band_energy: torch.Tensor
    band_multiplier: torch.Tensor
    ray_count: torch.Tensor
    order: torch.Tensor
    has_projection: torch.Tensor
    projection: torch.Tensor
    path_off: torch.Tensor
    path: torch.Tensor

    def __len__(self):
        return int(self.distance.numel())


# ---------------------------------------------------------------- CSR helpers
def _csr_gather(off: torch.Tensor, vals: torch.Tensor, perm: torch.Tensor):
    """Reorder CSR segments: segment perm[i] becomes segment i."""
    lens = (off[1:] - off[:-1])[perm]
    new_off = torch.zeros(len(perm) + 1, dtype=torch.int64, device=off.device)
    if len(perm):
        new_off[1:] = torch.cumsum(lens, 0)
    total = int(new_off[-1].item())
    if total == 0:
        return new_off, vals[:0]
    starts = off[:-1][perm]
    idx = torch.repeat_interleave(starts - new_off[:-1], lens) + torch.arange(total, device=off.device)
    return new_off, vals[idx]


def select(c: CaptureSet, mask: torch.Tensor) -> CaptureSet:
    """Captures where mask holds (e.g. one receiver of a multi-receiver trace)."""
    idx = torch.nonzero(mask).flatten()
    off, hist = _csr_gather(c.hist_off, c.hist, idx)
    return CaptureSet(c.ray[idx], c.point[idx], c.dir[idx], c.path[idx], c.mult[idx], off, hist)


def sort_reference_order(c: CaptureSet) -> CaptureSet:
    """Sort by (ray index, path length) as trace() leaves them
    (tracer.cpp:143-147).  A ray captures at most once per step and a step
    adds one face, so the path order of one ray's captures is its order."""
    if len(c) == 0:
        return c
    key = c.ray.to(torch.int64) * (1 << 21) + c.order
    perm = torch.sort(key, stable=True).indices
    off, hist = _csr_gather(c.hist_off, c.hist, perm)
    return CaptureSet(c.ray[perm], c.point[perm], c.dir[perm], c.path[perm], c.mult[perm], off, hist)


# ---------------------------------------------------------------- ownership
def order_counts(c: CaptureSet, max_order: int) -> torch.Tensor:
    """Captures per order 0..max_order (int64)."""
    return torch.bincount(c.order, minlength=max_order + 1)[: max_order + 1].to(torch.int64)


def assign_orders(counts: list[int], world: int) -> list[int]:
    """Deterministic LPT: order classes by decreasing count (ties: lower
    order first) to the least-loaded rank (ties: lower rank)."""
    owner = [0] * len(counts)
    load = [0] * world
    for o in sorted(range(len(counts)), key=lambda k: (-counts[k], k)):
        r = min(range(world), key=lambda q: (load[q], q))
        owner[o] = r
        load[r] += counts[o]
    return owner


def order_owners(c: CaptureSet, max_order: int, group=None) -> list[int]:
    """all_reduce of the order histogram, then assign_orders."""
    counts = order_counts(c, max_order)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, group=group)
        world = dist.get_world_size(group)
    else:
        world = 1
    return assign_orders([int(x) for x in counts.cpu().tolist()], world)


# ---------------------------------------------------------------- exchange
def _a2a(out_splits, in_splits, send: torch.Tensor, group, width: int = 1):
    """all_to_all_single of rows with `width` columns (uneven splits)."""
    shape = (sum(out_splits),) + tuple(send.shape[1:])
    recv = torch.empty(shape, dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send.contiguous(), out_splits, in_splits, group=group)
    return recv


def exchange_captures(c: CaptureSet, owner: list[int], group=None) -> CaptureSet:
    """Send every capture to the owner of its order class; returns the
    received captures in reference order (sort_reference_order)."""
    world = dist.get_world_size(group)
    dev = c.ray.device
    own = torch.tensor(owner, dtype=torch.int64, device=dev)
    lens = c.order
    dest = own[lens] if len(c) else torch.zeros(0, dtype=torch.int64, device=dev)
    perm = torch.sort(dest, stable=True).indices
    rec = torch.cat([c.ray.to(torch.float64)[:, None], lens.to(torch.float64)[:, None], c.point, c.dir,
                     c.path[:, None], c.mult], 1)[perm]
    _, hist = _csr_gather(c.hist_off, c.hist, perm)
    send_n = torch.bincount(dest, minlength=world).to(torch.int64)
    send_h = torch.zeros(world, dtype=torch.int64, device=dev)
    if len(c):
        send_h.index_add_(0, dest, lens)
    meta = torch.stack([send_n, send_h], 1)  # (world, 2)
    recv_meta = torch.empty_like(meta)
    dist.all_to_all_single(recv_meta, meta, group=group)
    in_n, in_h = send_n.cpu().tolist(), send_h.cpu().tolist()
    out_n, out_h = recv_meta[:, 0].cpu().tolist(), recv_meta[:, 1].cpu().tolist()
    r = _a2a(out_n, in_n, rec, group)
    h = _a2a(out_h, in_h, hist, group)
    m = r.shape[0]
    off = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    if m:
        off[1:] = torch.cumsum(r[:, 1].to(torch.int64), 0)
    got = CaptureSet(r[:, 0].to(torch.int64), r[:, 2:5].contiguous(), r[:, 5:8].contiguous(),
                     r[:, 8].contiguous(), r[:, 9:].contiguous(), off, h)
    return sort_reference_order(got)


def gather_images(im: ImageSet, group=None, dst: int = 0) -> ImageSet | None:
    """Image lists of all ranks to `dst`, ordered by order class (stable).
    Returns the merged set on dst, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = im.distance.device
    n = len(im)
    plen = (im.path_off[1:] - im.path_off[:-1]) if n else torch.zeros(0, dtype=torch.int64, device=dev)
    f = torch.float64
    rec = torch.cat([im.position, im.distance[:, None], im.band_energy, im.band_multiplier,
                     im.ray_count.to(f)[:, None], im.order.to(f)[:, None], im.has_projection.to(f)[:, None],
                     im.projection, plen.to(f)[:, None]], 1) if n else torch.zeros((0, IMG_FIELDS), dtype=f,
                                                                                   device=dev)
    send_n = [0] * world
    send_h = [0] * world
    send_n[dst] = n
    send_h[dst] = int(im.path_off[-1].item()) if n else 0
    meta = torch.tensor([[send_n[q], send_h[q]] for q in range(world)], dtype=torch.int64, device=dev)
    recv_meta = torch.empty_like(meta)
    dist.all_to_all_single(recv_meta, meta, group=group)
    out_n, out_h = recv_meta[:, 0].cpu().tolist(), recv_meta[:, 1].cpu().tolist()
    path = im.path[: send_h[dst]] if n else torch.zeros(0, dtype=torch.int32, device=dev)
    r = _a2a(out_n, send_n, rec, group)
    p = _a2a(out_h, send_h, path.to(torch.int32), group)
    if rank != dst:
        return None
    m = r.shape[0]
    off = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    if m:
        off[1:] = torch.cumsum(r[:, 26].to(torch.int64), 0)
    order = r[:, 21].to(torch.int32)
    perm = torch.sort(order.to(torch.int64), stable=True).indices
    off2, path2 = _csr_gather(off, p, perm)
    r = r[perm]
    return ImageSet(r[:, 0:3].contiguous(), r[:, 3].contiguous(), r[:, 4:12].contiguous(), r[:, 12:20].contiguous(),
                    r[:, 20].to(torch.int32), r[:, 21].to(torch.int32), r[:, 22].to(torch.int32),
                    r[:, 23:26].contiguous(), off2, path2)


def reduce_histogram(hist: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of the per-rank 8-band pulse histograms (NCCL all_reduce; on
    NVSwitch NCCL may reduce in the switch)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, group=group)
    return hist


# ---------------------------------------------------------------- GPU pipeline
def device_captures(dtrace, receiver: int | None = None) -> CaptureSet:
    """Captures of a device trace as CUDA tensors (device-to-device copy
    through rr_trace_captures)."""
    import ctypes as C

    from ._lib import check

    st = dtrace.stats
    n, th = int(st.n_captures), int(st.total_history)
    dev = torch.device("cuda", dtrace.tree.ctx.device)
    f = dict(dtype=torch.float64, device=dev)
    recv = torch.empty(n, dtype=torch.int32, device=dev)
    ray = torch.empty(n, dtype=torch.int32, device=dev)
    point, dirs = torch.empty((n, 3), **f), torch.empty((n, 3), **f)
    path, mult = torch.empty(n, **f), torch.empty((n, NUM_BANDS), **f)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    hist = torch.empty(max(th, 1), dtype=torch.int32, device=dev)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    check(dtrace.lib.rr_trace_captures(dtrace.h, vp(recv), vp(ray), vp(point), vp(dirs), vp(path), vp(mult),
                                       vp(off), vp(hist)))
    c = CaptureSet(ray.to(torch.int64), point, dirs, path, mult, off, hist[:th])
    if receiver is not None:
        c = select(c, recv == receiver)
    return c


def import_captures(tree, c: CaptureSet, receivers, receiver: int = 0):
    """rr_captures_import of a CaptureSet (device tensors) as receiver
    `receiver` of `receivers`; returns a DeviceTrace for K5."""
    import ctypes as C

    from . import _lib
    from .roomray import DeviceTrace

    recs = receivers if isinstance(receivers, (list, tuple)) else [receivers]
    rarr = (_lib.Receiver * len(recs))(*[_lib.Receiver((C.c_double * 3)(*map(float, r.center)), float(r.radius))
                                         for r in recs])
    n = len(c)
    recv = torch.full((max(n, 1),), receiver, dtype=torch.int32, device=c.ray.device)
    ray = c.ray.to(torch.int32).contiguous()
    hist = c.hist.to(torch.int32).contiguous() if c.hist.numel() else torch.zeros(1, dtype=torch.int32,
                                                                                  device=c.ray.device)
    ts = [recv, ray, c.point.contiguous(), c.dir.contiguous(), c.path.contiguous(), c.mult.contiguous(),
          c.hist_off.contiguous(), hist]
    vp = [C.c_void_p(t.data_ptr()) for t in ts]
    h = C.c_void_p()
    torch.cuda.synchronize(c.ray.device)  # torch's stream -> the library's stream
    _lib.check(tree.lib.rr_captures_import(tree.h, n, *vp, rarr, len(recs), C.byref(h)))
    return DeviceTrace(tree, h)


def images_to_tensors(dimages) -> ImageSet:
    """A device image set (rr_images) as CUDA tensors (D2D copies)."""
    import ctypes as C

    from ._lib import check

    n, tp = dimages.n, dimages.total_path
    dev = torch.device("cuda", torch.cuda.current_device())
    f = dict(dtype=torch.float64, device=dev)
    i = dict(dtype=torch.int32, device=dev)
    im = ImageSet(torch.empty((n, 3), **f), torch.empty(n, **f), torch.empty((n, NUM_BANDS), **f),
                  torch.empty((n, NUM_BANDS), **f), torch.empty(n, **i), torch.empty(n, **i), torch.empty(n, **i),
                  torch.empty((n, 3), **f), torch.empty(n + 1, dtype=torch.int64, device=dev),
                  torch.empty(max(tp, 1), **i))
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    check(dimages.lib.rr_images_get(dimages.h, vp(im.position), vp(im.distance), vp(im.band_energy),
                                    vp(im.band_multiplier), vp(im.ray_count), vp(im.order), vp(im.has_projection),
                                    vp(im.projection), vp(im.path_off), vp(im.path)))
    im.path = im.path[:tp]
    return im


@dataclass
class ShardedResult:
    """Per receiver r: images[r] (merged list, rank 0 only; None elsewhere),
    band_ir[r] (8, L) and broadband[r] (L,) on every rank."""

    images: list
    band_ir: list
    broadband: list
    ray_bounces: int             # this rank's
    local_images: int            # image sources built on this rank (all receivers)


def run_sharded(tree, source, receivers, config, *, air, options, sample_rate: float, length: int, taps: int = 1023,
                block: int = 4096, group=None, mark=None, exchange: bool | None = None,
                host: bool = False) -> ShardedResult:
    """trace -> exchange -> image sources -> IR for every receiver, the ranks
    of `group` each tracing a block-cyclic shard of the N-ray lattice (one
    trace serves all receivers: a receiver never alters a ray,
    tracer.cpp:27-29).  With a single rank it is the plain single-GPU
    pipeline.

    host=True returns the image lists and IRs in pinned host memory: a
    single rank's image list is copied to the host on a side stream while the
    IR stage runs on the context stream (the copy is PCIe bound, ~1 ms for
    C2's 56 MB, and the IR stage does not read it)."""
    import ctypes as C

    from . import _lib
    from .roomray import build_image_sources_device, trace_device

    recs = list(receivers) if isinstance(receivers, (list, tuple)) else [receivers]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shard = dict(first=rank, stride=world, block=block) if world > 1 else {}
    # exchange=True forces the collective path on one rank (tests)
    xch = world > 1 if exchange is None else bool(exchange)
    mark = mark or (lambda name: None)
    dt = trace_device(tree, source, recs, config, **shard)
    mark("trace")
    lib = tree.lib
    dev = torch.device("cuda", tree.ctx.device)
    out = ShardedResult([], [], [], int(dt.stats.ray_bounces), 0)
    caps_all = device_captures(dt) if xch else None
    recv_ids = None
    if xch:
        n = int(dt.stats.n_captures)
        recv_ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        _lib.check(lib.rr_trace_captures(dt.h, C.c_void_p(recv_ids.data_ptr()), None, None, None, None, None, None,
                                         None))
        recv_ids = recv_ids[:n]
    for r in range(len(recs)):
        if xch:
            caps = select(caps_all, recv_ids == r)
            owner = order_owners(caps, config.max_iterations, group)
            mine = exchange_captures(caps, owner, group)
            dt_local, ridx = import_captures(tree, mine, recs, r), r
            mark("exchange")
        else:
            dt_local, ridx = dt, r
        dimg = build_image_sources_device(dt_local, source.ray_count, air, options, receiver=ridx)
        mark("images")
        early = None
        if host and not xch:  # start the image list's D2H now, overlapping the IR stage
            early = images_to_host_async(dimg, dev)
            mark("gather")
        d_dist, d_en, n_img = dimg.device_arrays()
        hist = torch.empty(NUM_BANDS * (length + taps), dtype=torch.float64, device=dev)
        _lib.check(lib.rr_ir_bin_device(tree.ctx.h, n_img, C.c_void_p(d_dist), C.c_void_p(d_en),
                                        config.speed_of_sound, sample_rate, length + taps,
                                        C.c_void_p(hist.data_ptr())))
        # stream-level ordering only (a device-wide synchronize would also
        # wait for the side stream's image copy)
        _order(tree.ctx.stream, dev, ctx_first=True)
        reduce_histogram(hist, group)
        band = torch.empty(NUM_BANDS * length, dtype=torch.float64, device=dev)
        bb = torch.empty(length, dtype=torch.float64, device=dev)
        _order(tree.ctx.stream, dev, ctx_first=False)
        _lib.check(lib.rr_ir_filter_device(tree.ctx.h, C.c_void_p(hist.data_ptr()), sample_rate, taps, length,
                                           C.c_void_p(band.data_ptr()), C.c_void_p(bb.data_ptr())))
        _order(tree.ctx.stream, dev, ctx_first=True)
        mark("ir")
        if early is not None:
            local, side, _ = early  # (dimg stays referenced until the copy ran)
            out.local_images += len(local)
            out.images.append(local)
        else:
            local = images_to_tensors(dimg)
            out.local_images += len(local)
            merged = gather_images(local, group) if xch else local
            if host and merged is not None:
                merged, side = imageset_to_host_async(merged, dev, tree.ctx.stream)
                side.synchronize()
            out.images.append(merged)
        band = band.view(NUM_BANDS, length)
        if host:
            band, bb = _pinned_copy(band), _pinned_copy(bb)
        out.band_ir.append(band)
        out.broadband.append(bb)
        torch.cuda.synchronize(dev)
        mark("gather" if early is None else "host")
    return out


def _order(ctx_stream: int, dev, ctx_first: bool) -> None:
    """Make torch's current stream wait for the context stream (ctx_first)
    or the other way round."""
    if not ctx_stream:
        return
    ctx = torch.cuda.ExternalStream(ctx_stream, device=dev)
    cur = torch.cuda.current_stream(dev)
    a, b = (ctx, cur) if ctx_first else (cur, ctx)
    if a != b:
        ev = torch.cuda.Event()
        ev.record(a)
        b.wait_event(ev)


def _pinned_copy(t: torch.Tensor) -> torch.Tensor:
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h


def images_to_host_async(dimages, dev):
    """A device image set (rr_images) straight into pinned host tensors,
    copied on a side stream that starts after the image build
    (rr_images_get_async); returns (host set, stream, dimages).  The caller
    synchronizes the stream before reading the set or dropping dimages."""
    import ctypes as C

    from ._lib import check

    n, tp = dimages.n, dimages.total_path
    f = dict(dtype=torch.float64, pin_memory=True)
    i = dict(dtype=torch.int32, pin_memory=True)
    im = ImageSet(torch.empty((n, 3), **f), torch.empty(n, **f), torch.empty((n, NUM_BANDS), **f),
                  torch.empty((n, NUM_BANDS), **f), torch.empty(n, **i), torch.empty(n, **i), torch.empty(n, **i),
                  torch.empty((n, 3), **f), torch.empty(n + 1, dtype=torch.int64, pin_memory=True),
                  torch.empty(max(tp, 1), **i))
    side = torch.cuda.Stream(device=dev)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    check(dimages.lib.rr_images_get_async(dimages.h, C.c_void_p(side.cuda_stream), vp(im.position), vp(im.distance),
                                          vp(im.band_energy), vp(im.band_multiplier), vp(im.ray_count), vp(im.order),
                                          vp(im.has_projection), vp(im.projection), vp(im.path_off), vp(im.path)))
    im.path = im.path[:tp]
    return im, side, dimages


def imageset_to_host_async(im: ImageSet, dev, ctx_stream: int):
    """Copy a device ImageSet into pinned host tensors on a side stream that
    waits for the context stream's work so far; returns (host set, stream)."""
    ctx = torch.cuda.ExternalStream(ctx_stream, device=dev) if ctx_stream else torch.cuda.current_stream(dev)
    ready = torch.cuda.Event()
    ready.record(ctx)
    ready_cur = torch.cuda.Event()
    ready_cur.record(torch.cuda.current_stream(dev))  # torch.empty / D2D copies of images_to_tensors
    side = torch.cuda.Stream(device=dev)
    side.wait_event(ready)
    side.wait_event(ready_cur)
    with torch.cuda.stream(side):
        fields = {k: _pinned_copy(getattr(im, k)) for k in im.__dataclass_fields__}
    for k in im.__dataclass_fields__:  # the device tensors stay alive until the copy ran
        getattr(im, k).record_stream(side)
    return ImageSet(**fields), side
