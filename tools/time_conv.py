"""Time one conv pass with CUDA events: python tools/time_conv.py fprop|dgrad|wgrad N HW C K R stride pad"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32, ConvDesc  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402

kind = sys.argv[1]
n, hw, c, k, r, s, pad = (int(v) for v in sys.argv[2:9])
_lib.ctx.init(0)
lib, st = _lib.lib(), _lib.stream()
p = (hw + 2 * pad - r) // s + 1
d = ConvDesc(n, hw, hw, c, k, r, r, s, pad, p, p)
x, w, y = Buffer(n * hw * hw * c, BF16), Buffer(k * r * r * c, BF16), Buffer(n * p * p * k, BF16)
for t in (x, w, y):
    t.fill(0.01)
dw = Buffer(k * r * r * c, F32)
ws = Buffer(lib.nsk_conv2d_wgrad_workspace(C.byref(d)) // 4 + 1, F32)


def run():
    if kind == "fprop":
        return lib.nsk_conv2d_fprop(C.byref(d), x.ptr, w.ptr, y.ptr, 0, st)
    if kind == "dgrad":
        return lib.nsk_conv2d_dgrad(C.byref(d), y.ptr, w.ptr, x.ptr, st)
    return lib.nsk_conv2d_wgrad(C.byref(d), x.ptr, y.ptr, dw.ptr, 0.0, ws.ptr, ws.nbytes, st)


_lib.check(run())
e0, e1 = C.c_void_p(), C.c_void_p()
lib.nsk_event_create(1, C.byref(e0))
lib.nsk_event_create(1, C.byref(e1))
for _ in range(3):
    run()
lib.nsk_event_record(e0, st)
for _ in range(20):
    run()
lib.nsk_event_record(e1, st)
lib.nsk_event_sync(e1)
ms = C.c_float()
lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
us = ms.value * 50
print(f"{kind} n{n} {hw}x{hw} {c}->{k} {r}x{r} s{s} probe={os.environ.get('NSK_PROBE', '0')}: {us:.1f} us "
      f"{2.0 * n * p * p * k * c * r * r / us / 1e6:.0f} TFLOP/s")
