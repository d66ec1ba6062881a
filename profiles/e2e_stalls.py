"""Where the C5 end-to-end step loses time: the bench's e2e loop (scene from
pinned host arrays -> rr_pipeline_sharded -> results to host) repeated, with
the pipeline's own stage times per step, in three modes:
    pinned   outputs into page-locked arrays (bench.py's e2e)
    pageable outputs into numpy arrays
    device   image lists left on the device (IRs still fetched)
    python profiles/e2e_stalls.py <mode> [steps]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_05784_b200 import Context, Receiver, SourceConfig, TraceConfig, TriangleMesh, _lib, scenes  # noqa: E402
from paper_1811_05784_b200 import roomray as rr  # noqa: E402

mode = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
s = scenes.config5()
ctx = Context(0)
torch.cuda.synchronize()
pv = torch.from_numpy(s.vertices.reshape(-1)).pin_memory()
pt = torch.from_numpy(s.faces.reshape(-1)).pin_memory()
pa = torch.from_numpy(s.absorption.reshape(-1)).pin_memory()
lib = _lib.load()
mesh = TriangleMesh(s.vertices, s.faces, s.absorption)
L = int(round(s.ir_seconds * s.sample_rate))
dt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64}


def pinned(shape, dtype):
    return torch.empty(shape, dtype=dt[np.dtype(dtype)], pin_memory=True).numpy()


for it in range(steps):
    t0 = time.perf_counter()
    h = C.c_void_p()
    _lib.check(lib.rr_scene_create(ctx.h, C.c_void_p(pv.data_ptr()), len(s.vertices), C.c_void_p(pt.data_ptr()),
                                   len(s.faces), C.c_void_p(pa.data_ptr()), len(s.absorption), 1, C.byref(h)))
    t1 = time.perf_counter()
    sc = rr.AccelTree.__new__(rr.AccelTree)
    sc.ctx, sc.lib, sc.mesh, sc.h = ctx, lib, mesh, h
    res = rr.pipeline_sharded(sc, SourceConfig(s.source, s.ray_count), [Receiver(*r) for r in s.receivers],
                              TraceConfig(max_iterations=s.max_iterations, max_range=s.max_range),
                              options=rr.ClusterOptions(1e-6, True), sample_rate=s.sample_rate, length=L, taps=1023,
                              block=4096, device_images=(mode == "device"),
                              alloc=pinned if mode == "pinned" else np.empty)
    t2 = time.perf_counter()
    sm = res.stage_ms
    del res
    lib.rr_scene_destroy(h)
    sc.h = None
    t3 = time.perf_counter()
    print(f"{mode} step {it}: scene {1e3 * (t1 - t0):7.1f}  pipeline+fetch {1e3 * (t2 - t1):7.1f}  "
          f"free {1e3 * (t3 - t2):6.1f} ms | " + " ".join(f"{k} {v:.1f}" for k, v in sm.items()), flush=True)
