"""C4 IR-synthesis timing (development tool): bin + FIR of 2M image sources."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1811_05784_b200 import roomray as rr, scenes, _lib  # noqa: E402

c4 = scenes.config4()
ctx = rr.Context.default(0)
n = len(c4["distance"])
L = int(round(c4["seconds"] * c4["sample_rate"]))
taps = c4["taps"]
d = torch.from_numpy(c4["distance"]).cuda()
e = torch.from_numpy(c4["energy"].reshape(-1)).cuda()
hist = torch.empty(8 * (L + taps), dtype=torch.float64, device="cuda")
band = torch.empty(8 * L, dtype=torch.float64, device="cuda")
bb = torch.empty(L, dtype=torch.float64, device="cuda")
st = torch.cuda.ExternalStream(ctx.stream)
for it in range(5):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    with torch.cuda.stream(st):
        e0.record()
    _lib.check(ctx.lib.rr_ir_bin_device(ctx.h, n, C.c_void_p(d.data_ptr()), C.c_void_p(e.data_ptr()), 343.0,
                                        c4["sample_rate"], L + taps, C.c_void_p(hist.data_ptr())))
    with torch.cuda.stream(st):
        e1.record()
    _lib.check(ctx.lib.rr_ir_filter_device(ctx.h, C.c_void_p(hist.data_ptr()), c4["sample_rate"], taps, L,
                                           C.c_void_p(band.data_ptr()), C.c_void_p(bb.data_ptr())))
    with torch.cuda.stream(st):
        e2.record()
    torch.cuda.synchronize()
    print(f"bin {e0.elapsed_time(e1):.3f} ms  fir {e1.elapsed_time(e2):.3f} ms", file=sys.stderr)
t = time.perf_counter()
out = rr.synthesize(c4["distance"], c4["energy"], 343.0, c4["sample_rate"], taps=taps, length=L)
print(f"host-to-host synthesize {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr)
