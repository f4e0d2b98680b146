"""A/B a libnskb environment switch on selected conv passes, interleaved in one process (medians of rounds).

    python tools/ab_conv.py NSK_CONV_RR 0 1 [resnet18|resnet50] [batch]
"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import conv_table as T  # noqa: E402

from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32, ConvDesc  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402


def main():
    var, va, vb = sys.argv[1:4]
    model = sys.argv[4] if len(sys.argv) > 4 else "resnet18"
    b = int(sys.argv[5]) if len(sys.argv) > 5 else 256
    _lib.ctx.init(0)
    lib, st = _lib.lib(), _lib.stream()
    convs = T.resnet18_convs(b) if model == "resnet18" else T.resnet50_convs(b)
    e0, e1 = C.c_void_p(), C.c_void_p()
    lib.nsk_event_create(1, C.byref(e0))
    lib.nsk_event_create(1, C.byref(e1))
    tot = {va: 0.0, vb: 0.0}
    for (n, hw, c, k, r, s, pad), cnt in sorted(convs.items()):
        p = (hw + 2 * pad - r) // s + 1
        d = ConvDesc(n, hw, hw, c, k, r, r, s, pad, p, p)
        x, w, y = Buffer(n * hw * hw * c, BF16), Buffer(k * r * r * c, BF16), Buffer(n * p * p * k, BF16)
        for t in (x, w, y):
            t.fill(0.01)
        dw = Buffer(k * r * r * c, F32)
        ws = Buffer(lib.nsk_conv2d_wgrad_workspace(C.byref(d)) // 4 + 1, F32)
        for kind in ("fprop", "dgrad", "wgrad"):
            def run():
                if kind == "fprop":
                    return lib.nsk_conv2d_fprop(C.byref(d), x.ptr, w.ptr, y.ptr, 0, st)
                if kind == "dgrad":
                    return lib.nsk_conv2d_dgrad(C.byref(d), y.ptr, w.ptr, x.ptr, st)
                return lib.nsk_conv2d_wgrad(C.byref(d), x.ptr, y.ptr, dw.ptr, 0.0, ws.ptr, ws.nbytes, st)
            res = {va: [], vb: []}
            for rnd in range(5):
                for v in (va, vb):
                    os.environ[var] = v
                    run()
                    lib.nsk_event_record(e0, st)
                    for _ in range(10):
                        run()
                    lib.nsk_event_record(e1, st)
                    lib.nsk_event_sync(e1)
                    ms = C.c_float()
                    lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
                    res[v].append(100.0 * ms.value)
            ma, mb = statistics.median(res[va]), statistics.median(res[vb])
            tot[va] += ma * cnt
            tot[vb] += mb * cnt
            print(f"{kind:5s} {hw:3d}x{hw:<3d} {c:4d}->{k:4d} {r}x{r} s{s} x{cnt}: {var}={va} {ma:7.1f} us  "
                  f"{var}={vb} {mb:7.1f} us  ({100 * (ma - mb) / ma:+.1f}%)", flush=True)
    print(f"TOTAL {var}={va} {tot[va]:.1f} us   {var}={vb} {tot[vb]:.1f} us")


if __name__ == "__main__":
    main()
