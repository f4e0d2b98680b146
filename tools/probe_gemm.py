"""Time nsk_gemm (bf16, K-major) on conv-like shapes: is the 4D conv feed or the kernel itself the limit?"""
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
for (M, N, K) in [(262144, 64, 576), (65536, 128, 1152), (16384, 256, 2304), (8192, 8192, 8192), (262144, 64, 64),
                  (65536, 256, 4096)]:
    a = Buffer(M * K, BF16)
    a.fill(0.01)
    b = Buffer(N * K, BF16)
    b.fill(0.01)
    c = Buffer(M * N, BF16)
    for _ in range(3):
        _lib.check(lib.nsk_gemm(BF16, 0, 0, M, N, K, a.ptr, K, b.ptr, K, c.ptr, N, 0, None, 0.0, st))
    e0, e1 = C.c_void_p(), C.c_void_p()
    lib.nsk_event_create(1, C.byref(e0))
    lib.nsk_event_create(1, C.byref(e1))
    lib.nsk_event_record(e0, st)
    it = 10
    for _ in range(it):
        lib.nsk_gemm(BF16, 0, 0, M, N, K, a.ptr, K, b.ptr, K, c.ptr, N, 0, None, 0.0, st)
    lib.nsk_event_record(e1, st)
    lib.nsk_event_sync(e1)
    ms = C.c_float()
    lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
    t = ms.value / it
    print(f"gemm M={M} N={N} K={K}: {t*1000:.1f} us  {2*M*N*K/t/1e9:.0f} TFLOP/s", flush=True)
