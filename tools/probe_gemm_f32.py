"""Time the fp32-output GEMM with bias (the GRU input projection, 8192 x 1536 x 512) alone: NSK_PROBE=1 skips the
MMAs, 2 the stores (diagnostics)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402

_lib.ctx.init(0)
lib = _lib.lib()
st = _lib.stream()
M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 1536, 512)))
a = Buffer(M * K, BF16)
a.fill(0.01)
b = Buffer(N * K, BF16)
b.fill(0.01)
bias = Buffer(N, F32)
bias.fill(0.5)
c = Buffer(M * N, F32)
run = lambda: lib.nsk_gemm(BF16, 0, 0, M, N, K, a.ptr, K, b.ptr, K, c.ptr, N, 1, C.c_void_p(bias.ptr), 0.0, st)  # noqa
for _ in range(3):
    _lib.check(run())
e0, e1 = C.c_void_p(), C.c_void_p()
lib.nsk_event_create(1, C.byref(e0))
lib.nsk_event_create(1, C.byref(e1))
it = 20
lib.nsk_event_record(e0, st)
for _ in range(it):
    run()
lib.nsk_event_record(e1, st)
_lib.sync()
ms = C.c_float()
lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
us = ms.value * 1000 / it
print(f"gemm f32 {M}x{N}x{K} probe={os.environ.get('NSK_PROBE', '0')}: {us:.1f} us, "
      f"{2 * M * N * K / us / 1e6:.0f} TFLOP/s, out {M * N * 4 / us / 1e3:.0f} GB/s")
