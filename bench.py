"""Benchmark: rays*bounces/s of the specular trace on B200 (BASELINE.json
metric), with the HBM-roofline fraction and the reference CPU path beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
                  [--impl ours|reference] [--dry-run]

Workload (config.workload): BASELINE.json configs[4] (C5), the config the
metric is quoted on ("rays sharded over 1/2/4/8 B200") — a 30x20x12 m room
filled with 500 seeded rotated icosphere and box scatterers, 2 000 000
triangles, seeded per-octave absorption, 8 * 10^6 Fibonacci rays, 100
reflections; 3 s IR at 48 kHz.  Synthetic, seeded (the reference ships no
such mesh).  It is the only HBM-resident scene (C1-C3 fit in the 126 MB L2).
--config c1/c2/c3 run the other traced configs.

One step = one trace of the whole lattice (device emission, persistent
traversal kernel, capture compaction + sort) on the device-resident scene:
`value` counts the nearest-hit queries executed (ray*bounces) per second.
`e2e` is the same metric through the C ABI from pinned host arrays, every
step: scene upload + device validation + tree build (rr_scene_create), then
rr_pipeline_sharded -- trace, the NCCL capture exchange when N > 1, image
sources (coplanar merge on, RunConfig default), exact multi-GPU 8-band IR --
and the download of every image list and IR.  `e2e_native_cpp` times the C++
facade's run_trace_pipeline stages (tests/native/pipeline_bench.cpp).

Multi-GPU: strong scaling of the fixed 8 * 10^6-ray lattice, each rank
tracing a block-cyclic shard (4 096-ray blocks), time = max over ranks.
`--gpus N` without a torchrun environment re-launches this script under
torch.distributed.run with N ranks (127.0.0.1); `--dry-run` does the same
with gloo on CPU and no kernels (launcher and reduction check).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rays*bounces/sec (and % of HBM roofline)"
UNIT = "ray*bounces/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
BRB_FILE = os.path.join(ROOT, "profiles", "brb_frozen.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def brb_model(config):
    with open(BRB_FILE) as f:
        return json.load(f)[config]


UNIT_SCALE = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
              "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def ncu_trace_counters(config):
    """Per-launch DRAM / L2 bytes and duration of the trace kernel from the
    committed raw ncu export profiles/ncu_trace_<config>.csv (`ncu --metrics
    dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,
    gpu__time_duration.sum -k regex:trace_kernel --csv --page raw`, the
    command is in the file's sibling .cmd).  None when absent."""
    import csv
    path = os.path.join(ROOT, "profiles", f"ncu_trace_{config}.csv")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        rows = [r for r in csv.reader(f) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    names, units = rows[head], rows[head + 1]
    want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum")
    opt = ("smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__thread_inst_executed_per_inst_executed.ratio")
    col = {w: names.index(w) for w in want}
    col.update({w: names.index(w) for w in opt if w in names})
    kcol = names.index("Kernel Name")
    acc = {w: [] for w in col}
    for r in rows[head + 2:]:
        if len(r) != len(names) or "trace_kernel" not in r[kcol]:
            continue
        for w in col:
            scale = UNIT_SCALE.get(units[col[w]].lower(), 1.0) if w in want else 1.0
            acc[w].append(float(r[col[w]].replace(",", "")) * scale)
    if not acc[want[0]]:
        return None
    mean = {w: sum(v) / len(v) for w, v in acc.items()}
    out = {"dram_bytes": mean[want[0]] + mean[want[1]], "dram_read": mean[want[0]], "dram_write": mean[want[1]],
           "l2_bytes": mean[want[2]], "ncu_ms": mean[want[3]] * 1e3, "launches": len(acc[want[0]]),
           "source": os.path.relpath(path, ROOT)}
    if opt[0] in mean:
        out.update({"warp_inst": mean[opt[0]], "issue_active_pct": mean.get(opt[1]),
                    "threads_per_inst": mean.get(opt[2])})
    return out


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every 10 ms through NVML while
    the timed region runs (nvidia-smi's 200 ms loop would miss a short
    region)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device):
        self.device = device
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.sm.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                bits = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS:
                    if bits & getattr(N, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __exit__(self, *a):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


# ---------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_scene(name):
    from paper_1811_05784_b200 import scenes
    return scenes.CONFIGS[name]()


def cpu_reference_sample(scene, seconds, threads, stride=None):
    """The reference's own trace loop (oracle/_ref: unmodified tracer.cpp,
    step() with thread_count = threads) on a strided subset of the lattice,
    sized to ~`seconds` of work (or the given stride).  Returns (rate,
    sample description, kind, ray*bounces, seconds, stride)."""
    import oracle
    if oracle.ref_available():
        lib = oracle.Ref()
        sc = lib.scene(oracle.Mesh(scene.vertices, scene.faces, scene.absorption))
        kind = "reference"

        def run(stride):
            t = time.perf_counter()
            _, st = sc.trace(scene.source, scene.ray_count, scene.receivers[0][0], scene.receivers[0][1],
                             scene.max_iterations, scene.max_range, threads, 0, stride, 0)
            return st.ray_bounces, time.perf_counter() - t
    else:
        lib = oracle.Port()
        sc = lib.scene(oracle.Mesh(scene.vertices, scene.faces, scene.absorption))
        kind = "port"

        def run(stride):
            t = time.perf_counter()
            _, st = sc.trace(scene.source, scene.ray_count, [scene.receivers[0][0]], [scene.receivers[0][1]],
                             scene.max_iterations, scene.max_range, threads, 0, stride, 0)
            return st.ray_bounces, time.perf_counter() - t
    # size the strided sample to ~`seconds` (the first probes underestimate
    # the rate: thread start-up and tail imbalance on few rays)
    fixed = stride is not None
    stride = stride if fixed else max(1, scene.ray_count // 2000)
    rb, dt = run(stride)
    for _ in range(0 if fixed else 3):
        if dt >= 0.5 * seconds or stride == 1:
            break
        rays_now = (scene.ray_count + stride - 1) // stride
        want = rays_now * seconds / max(dt, 1e-3)
        stride = max(1, int(scene.ray_count // max(want, 1)))
        rb, dt = run(stride)
    rays = (scene.ray_count + stride - 1) // stride
    return rb / dt, f"{rays} of {scene.ray_count} lattice rays (k = 0 mod {stride}), {rb} ray*bounces, {dt:.2f} s", \
        kind, rb, dt, stride


def write_scene_bin(scene, path):
    """The scene as tests/native/pipeline_bench.cpp reads it (receiver 0)."""
    (c, r), = scene.receivers[:1]
    with open(path, "wb") as f:
        f.write(np.array([len(scene.vertices), len(scene.faces), len(scene.absorption)], np.int64).tobytes())
        f.write(np.ascontiguousarray(scene.vertices, np.float64).tobytes())
        f.write(np.ascontiguousarray(scene.faces, np.int32).tobytes())
        f.write(np.ascontiguousarray(scene.absorption, np.float64).tobytes())
        f.write(np.array(scene.source, np.float64).tobytes())
        f.write(np.array([scene.ray_count], np.int64).tobytes())
        f.write(np.array([*c, r, scene.max_range, scene.sample_rate], np.float64).tobytes())
        f.write(np.array([scene.max_iterations, 1], np.int64).tobytes())


def native_pipeline(scene, steps, warmup):
    """The C++ facade's run_trace_pipeline stages (tests/native/pipeline_bench.cpp:
    tree build, trace, image sources, pulse trains + IR, factors; host mesh
    in, host artifacts out), compiled here with g++ against the library."""
    import tempfile
    exe = os.path.join(ROOT, "build", "pipeline_bench")
    src = os.path.join(ROOT, "tests", "native", "pipeline_bench.cpp")
    lib_dir = os.path.join(ROOT, "paper_1811_05784_b200")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-L", lib_dir,
                    "-lroomray_b200", "-Wl,-rpath," + lib_dir, "-o", exe], check=True)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "scene.bin")
        write_scene_bin(scene, path)
        out = subprocess.run([exe, path, str(steps), str(warmup)], capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh
    from paper_1811_05784_b200 import roomray as rr
    from paper_1811_05784_b200 import _lib

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    scene = load_scene(args.config)
    ctx = Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    mesh = TriangleMesh(scene.vertices, scene.faces, scene.absorption)
    tree = rr.AccelTree(mesh, ctx)
    n_total = scene.ray_count  # strong scaling: the config's lattice split over the ranks
    src = SourceConfig(scene.source, n_total)
    recv = [Receiver(*r) for r in scene.receivers]
    cfg = TraceConfig(max_iterations=scene.max_iterations, max_range=scene.max_range)
    shard = dict(first=rank, stride=world, block=4096) if world > 1 else {}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def one_trace():
        return rr.trace_device(tree, src, recv, cfg, **shard)

    barrier()  # (NCCL communicator created here for N > 1)
    nccl = nccl_init_lines() if world > 1 and rank == 0 else None
    for _ in range(args.warmup):
        one_trace()
    # ---- timed: device-resident trace
    step_ms, kern_ms, bounces, launches = [], [], 0, 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush (512 MB > 126 MB L2) between steps
            barrier()
            l0 = ctx.launches
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record()
            dt = one_trace()
            with torch.cuda.stream(stream):
                e1.record()
            barrier()
            step_ms.append(e0.elapsed_time(e1))
            kern_ms.append(dt.kernel_ms)
            bounces += dt.stats.ray_bounces
            launches += ctx.launches - l0
            del dt
    my_ms = sum(step_ms)
    t = torch.tensor([my_ms, float(bounces)], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_ms, total_bounces = tmax[0].item(), tsum[1].item()
    else:
        total_ms, total_bounces = my_ms, float(bounces)
    value = total_bounces / (total_ms / 1e3)

    # ---- e2e through the C ABI from pinned host buffers
    pv = torch.from_numpy(scene.vertices.reshape(-1)).pin_memory()
    pt = torch.from_numpy(scene.faces.reshape(-1)).pin_memory()
    pa = torch.from_numpy(scene.absorption.reshape(-1)).pin_memory()
    L = int(round(scene.ir_seconds * scene.sample_rate))
    taps = 1023
    h2d = pv.numel() * 8 + pt.numel() * 4 + pa.numel() * 8
    e2e_ms, d2h, breakdown = [], 0, {}

    lib = _lib.load()
    import ctypes as C

    # the multi-GPU pipeline behind the C ABI (rr_pipeline_sharded): its own
    # NCCL communicator, the unique id from rank 0 over torch.distributed
    _torch_dt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32,
                 np.dtype(np.int64): torch.int64}

    def pinned(shape, dtype):  # page-locked host outputs (full PCIe bandwidth)
        return torch.empty(shape, dtype=_torch_dt[np.dtype(dtype)], pin_memory=True).numpy()

    comm = None
    if world > 1:
        uid = [rr.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = rr.Comm(ctx, uid[0], world, rank)
    for it in range(args.warmup + args.steps):
        barrier()
        w0 = time.perf_counter()
        e0, e1, e_sc = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        with torch.cuda.stream(stream):
            e0.record()
        h = C.c_void_p()
        _lib.check(lib.rr_scene_create(ctx.h, C.c_void_p(pv.data_ptr()), len(scene.vertices),
                                       C.c_void_p(pt.data_ptr()), len(scene.faces), C.c_void_p(pa.data_ptr()),
                                       len(scene.absorption), 1, C.byref(h)))
        with torch.cuda.stream(stream):
            e_sc.record()
        sc = rr.AccelTree.__new__(rr.AccelTree)
        sc.ctx, sc.lib, sc.mesh, sc.h = ctx, lib, mesh, h
        res = rr.pipeline_sharded(sc, src, recv, cfg, comm=comm, air=rr.AirModel(),
                                  options=rr.ClusterOptions(1e-6, True), sample_rate=scene.sample_rate, length=L,
                                  taps=taps, block=4096, alloc=pinned)
        # results in host memory: every receiver's 8 band IRs and broadband IR
        # (every rank), the merged image list (rank 0)
        fetched = []
        for r, band in enumerate(res.band_ir):
            fetched += [band, res.broadband[r]]
            im = res.images[r]
            fetched += [getattr(im, f) for f in im.__dataclass_fields__]
        with torch.cuda.stream(stream):
            e1.record()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        if it >= args.warmup:
            e2e_ms.append(max(e0.elapsed_time(e1), (w1 - w0) * 1e3))
            stages = {"scene": e0.elapsed_time(e_sc), **res.stage_ms}
            stages["fetch+host"] = e2e_ms[-1] - sum(stages.values())
            for k, v in stages.items():
                breakdown[k] = breakdown.get(k, 0.0) + v / args.steps
            d2h = sum(np.asarray(x).nbytes for x in fetched)
        del res
        lib.rr_scene_destroy(h)
        sc.h = None
        if os.environ.get("RR_E2E_DEBUG"):
            from cuda.bindings import runtime as crt
            _, pool = crt.cudaDeviceGetDefaultMemPool(local)
            _, rsv = crt.cudaMemPoolGetAttribute(pool, crt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
            _, used = crt.cudaMemPoolGetAttribute(pool, crt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemHigh)
            print(f"e2e dbg step {it}: {e2e_ms[-1] if it >= args.warmup else 0:.1f} ms, pool reserved "
                  f"{int(rsv) / 2**30:.2f} GiB, used high {int(used) / 2**30:.2f} GiB", file=sys.stderr)
    del comm
    e2e_local = sum(e2e_ms)
    t = torch.tensor([e2e_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = total_bounces / (t.item() / 1e3)

    # ---- roofline of the dominant kernel (trace_kernel)
    # primary: the kernel's MEASURED DRAM bytes per launch (committed raw ncu
    # export of this config) over its live launch time in this run; the
    # reference-tree byte model and the kernel's own work model
    # are reported beside it
    model = brb_model(args.config)
    peak, peak_kind = hbm_peak()
    kern_s = sum(kern_ms) / 1e3
    kern_ms_launch = 1e3 * kern_s / args.steps
    ncu = ncu_trace_counters(args.config)
    # the byte models on the work this kernel actually does (SAH tree,
    # conservative boxes, coplanar culling): one instrumented, untimed trace
    cnt = rr.trace_device(tree, src, recv, cfg, flags=_lib.RR_TRACE_COUNT, **shard).stats
    b_bar = cnt.ray_bounces / max(cnt.n_rays, 1)
    v_rb, l_rb = cnt.node_visits / cnt.ray_bounces, cnt.leaf_tests / cnt.ray_bounces
    b_kernel = cnt.node_bytes * v_rb + 80 * l_rb + 48 + 4 + 128 / b_bar
    ref_model_gbs = model["B_rb"] * bounces / kern_s / 1e9
    l2 = C.c_double()
    _lib.check(lib.rr_l2_read_gbs(ctx.h, 48 << 20, 40, C.byref(l2)))
    roof = {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_kind,
            "kernel_ms_per_launch": round(kern_ms_launch, 3),
            "kernel_share_of_step": round(sum(kern_ms) / my_ms, 3)}
    if ncu is not None and world == 1:
        achieved = ncu["dram_bytes"] / (kern_ms_launch / 1e3) / 1e9
        roof.update({"achieved": round(achieved, 1), "frac": round(achieved / peak, 4),
                     "traffic": round(ncu["dram_bytes"]), "basis": "ncu-measured DRAM bytes per launch "
                     "(dram__bytes_read.sum + dram__bytes_write.sum, " + ncu["source"] + ") / live kernel time",
                     "traffic_per_ray_bounce": round(ncu["dram_bytes"] / (bounces / args.steps), 1),
                     "l2_bytes_per_launch": round(ncu["l2_bytes"]),
                     "l2_achieved": round(ncu["l2_bytes"] / (kern_ms_launch / 1e3) / 1e9, 1),
                     "ncu_ms_per_launch": round(ncu["ncu_ms"], 3)})
        if ncu.get("issue_active_pct") is not None:
            # what does bound the kernel: the SM issue slots (ncu, same capture)
            busy = ncu["issue_active_pct"] >= 65.0
            roof["limiter"] = {"what": "SM instruction issue (not DRAM bandwidth)" if busy else
                               "latency of dependent node fetches (issue slots idle, not DRAM bandwidth)",
                               "issue_active_frac": round(ncu["issue_active_pct"] / 100.0, 4),
                               "warp_instructions_per_launch": round(ncu["warp_inst"]),
                               "threads_per_instruction": round(ncu["threads_per_inst"], 2)}
    else:
        roof.update({"achieved": None, "frac": None, "traffic": None,
                     "basis": "no committed ncu export for this config / world size"})
    roof["model"] = {
        "reference_tree_bytes_per_rb": round(model["B_rb"], 1),
        "reference_tree_equiv_gbs": round(ref_model_gbs, 1),
        "reference_tree_equiv_frac": round(ref_model_gbs / peak, 4),
        "note": "SURVEY 8(d) B_rb prices the reference median tree's node visits (n_int, n_leaf counted by the "
                "oracle); the SAH/wide traversal here visits fewer nodes, so this is a throughput equivalent",
        "kernel_tree_width": cnt.tree_width, "kernel_node_bytes": cnt.node_bytes,
        "kernel_node_visits_per_rb": round(v_rb, 2), "kernel_leaf_tests_per_rb": round(l_rb, 2),
        "kernel_bytes_per_rb": round(b_kernel, 1),
        "kernel_equiv_gbs": round(b_kernel * bounces / kern_s / 1e9, 1),
        "l2_peak_measured": round(l2.value, 1)}

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            rate, sample, kind, _, _, _ = cpu_reference_sample(scene, args.cpu_seconds, threads)
            cpu = {"value": round(rate, 1), "unit": UNIT, "cores": threads, "kind": kind, "sample": sample}
        native = None
        if world == 1 and not args.no_native:
            nat = native_pipeline(scene, max(2, args.steps // 3), 1)
            native = {"value": round(nat["ray_bounces_per_step"] / nat["seconds_per_step"], 1), "unit": UNIT,
                      "seconds_per_step": nat["seconds_per_step"], "stage_s": nat["stage_s"], "steps": nat["steps"],
                      "images": nat["images"], "captures": nat["captures"],
                      "what": "C++ facade run_trace_pipeline stages (tree build .. factors), host mesh in, host "
                              "artifacts out (captures, images, pulse trains, IR, factors), wall clock"}
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (fp32 conservative box filter)",
            "data": "synthetic (seeded splitmix64 scene; no dataset)",
            "config": bench_config(args, scene),
            "run": {"rays_per_gpu": -(-scene.ray_count // world), "parallelism": f"rays block-cyclic x{world}",
                    "l2": "flushed between timed steps (512 MB write)"},
            "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": round(t.item() / args.steps, 3),
                    "stage_ms": {k: round(v, 3) for k, v in breakdown.items()}},
            "e2e_native_cpp": native,
            "roofline": roof, "cpu_baseline": cpu, "gpu_launches": int(launches), "nccl": nccl,
            "clocks": clk.summary(),
            "ray_bounces_per_step": int(total_bounces / args.steps),
        }
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def bench_config(args, scene):
    """The workload both arms report (identical dicts, so the driver can
    match the lines); how each arm ran it goes under "run"."""
    return {"workload": f"{args.config}: {scene.name}, {scene.n_faces} tri, {scene.ray_count} rays, "
                        f"{scene.max_iterations} refl, {len(scene.receivers)} receiver(s)",
            "l2": "GPU arm: flushed between timed steps (512 MB write); CPU arm: n/a"}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    scene = load_scene(args.config)
    threads = os.cpu_count() or 1
    # the sample size (lattice stride) is fixed once, ~cpu_seconds / 2 of
    # work per step; every step then traces that same subset
    per_step = max(2.0, args.cpu_seconds / 2)
    stride = None
    rates = []
    for i in range(args.warmup + args.steps):
        rate, sample, kind, rb, dt, stride = cpu_reference_sample(scene, per_step, threads, stride)
        if i >= args.warmup:
            rates.append((rb, dt, sample, kind))
    rb = sum(r[0] for r in rates)
    dt = sum(r[1] for r in rates)
    value = rb / dt
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
           "data": "synthetic (seeded splitmix64 scene; no dataset)",
           "config": bench_config(args, scene), "run": {"parallelism": f"{threads} CPU threads"},
           "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": threads, "kind": rates[0][3],
                            "sample": rates[0][2] + " per step"},
           "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return out


def nccl_init_lines():
    """NCCL_DEBUG=INFO init lines of this process (launch() routes them to
    NCCL_DEBUG_FILE): the communicator's rank count as NCCL saw it."""
    import glob
    import re
    pat = os.environ.get("NCCL_DEBUG_FILE")
    if not pat:
        return None
    path = pat.replace("%h", "*").replace("%p", str(os.getpid()))
    for fn in glob.glob(path):
        with open(fn, errors="replace") as f:
            txt = f.read()
        m = re.findall(r"nRanks (\d+)", txt)
        ver = re.search(r"NCCL version ([\w.+-]+)", txt)
        return {"nRanks": int(m[-1]) if m else None, "version": ver.group(1) if ver else None, "log": fn}
    return None


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch(args):
    """--gpus N outside torchrun: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous)."""
    env = dict(os.environ)
    if not args.dry_run:
        # NCCL's init lines (rank count, transport) go to a per-rank file;
        # rank 0 reports the communicator size it saw in the JSON line
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", os.path.join("/tmp", "rr_bench_nccl.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """Launcher / reduction check without a GPU: every rank derives its
    block-cyclic shard of the lattice exactly as run_trace does, the counts
    are summed and a per-rank time max-reduced over gloo, rank 0 prints."""
    import torch
    import torch.distributed as dist

    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    scene = load_scene(args.config)
    n, block = scene.ray_count, 4096
    nblk = (n + block - 1) // block
    mine = sum(min(n, (b + 1) * block) - b * block for b in range(rank, nblk, world))
    t = torch.tensor([float(mine), float(rank + 1)], dtype=torch.float64)
    tot = t.clone()
    mx = t.clone()
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "rays_total": int(tot[0].item()),
                          "rays_rank0": mine, "lattice": n, "max_over_ranks": mx[1].item(),
                          "scaling": "strong", "config": {"workload": args.config}}))
        assert int(tot[0].item()) == n
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-native", action="store_true", help="skip the C++ facade pipeline timing")
    ap.add_argument("--dry-run", action="store_true", help="gloo/CPU launcher check, no kernels")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
