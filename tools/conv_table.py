"""Per-layer conv timing table: every distinct conv pass of a model, timed alone with CUDA events.

    python tools/conv_table.py [resnet18|resnet50] [batch]

Prints one line per (shape, pass): count in the model, us per launch, TFLOP/s, and the model-weighted
total, so the dominant passes are obvious. Not a bench number (kernels timed back to back, warm L2). Random
operands (CONST=1: the constant ones earlier tables used, which flatter the tensor pipe).
"""
import collections
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32, ConvDesc  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402


def resnet18_convs(b):
    out = collections.Counter()
    h, cin = 32, 64
    for cout, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
        for i in range(2):
            st = stride if i == 0 else 1
            out[(b, h, cin, cout, 3, st, 1)] += 1
            ho = h // st
            out[(b, ho, cout, cout, 3, 1, 1)] += 1
            if st != 1 or cin != cout:
                out[(b, h, cin, cout, 1, st, 0)] += 1
            h, cin = ho, cout
    return out


def resnet50_convs(b):
    out = collections.Counter()
    h, cin = 56, 64
    for width, blocks, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
        cout = width * 4
        for i in range(blocks):
            st = stride if i == 0 else 1
            out[(b, h, cin, width, 1, 1, 0)] += 1
            out[(b, h, width, width, 3, st, 1)] += 1
            ho = h // st
            out[(b, ho, width, cout, 1, 1, 0)] += 1
            if i == 0:
                out[(b, h, cin, cout, 1, st, 0)] += 1
            h, cin = ho, cout
    return out


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    iters = int(os.environ.get("ITERS", "20"))
    _lib.ctx.init(0)
    lib = _lib.lib()
    st = _lib.stream()
    convs = resnet18_convs(b) if model == "resnet18" else resnet50_convs(b)
    e0, e1 = C.c_void_p(), C.c_void_p()
    lib.nsk_event_create(1, C.byref(e0))
    lib.nsk_event_create(1, C.byref(e1))
    grand = 0.0
    gflop = 0.0
    rows = []
    rng = np.random.default_rng(0)
    for (n, hw, c, k, r, s, pad), cnt in sorted(convs.items()):
        p = (hw + 2 * pad - r) // s + 1
        d = ConvDesc(n, hw, hw, c, k, r, r, s, pad, p, p)
        x = Buffer(n * hw * hw * c, BF16)
        w = Buffer(k * r * r * c, BF16)
        y = Buffer(n * p * p * k, BF16)
        if os.environ.get("CONST") == "1":  # constant operands (understate the tensor pipe's power draw)
            x.fill(0.25)
            w.fill(0.01)
            y.fill(0.5)
        else:
            x.upload(rng.standard_normal(x.capacity).astype(np.float32))
            w.upload((rng.standard_normal(w.capacity) / np.sqrt(r * r * c)).astype(np.float32))
            y.upload(rng.standard_normal(y.capacity).astype(np.float32))
        dw = Buffer(k * r * r * c, F32)
        ws_b = lib.nsk_conv2d_wgrad_workspace(C.byref(d))
        ws = Buffer(ws_b // 4 + 1, F32)
        flops = 2.0 * n * p * p * k * c * r * r
        for kind in ("fprop", "dgrad", "wgrad"):
            def run():
                if kind == "fprop":
                    return lib.nsk_conv2d_fprop(C.byref(d), x.ptr, w.ptr, y.ptr, 0, st)
                if kind == "dgrad":
                    return lib.nsk_conv2d_dgrad(C.byref(d), y.ptr, w.ptr, x.ptr, st)
                return lib.nsk_conv2d_wgrad(C.byref(d), x.ptr, y.ptr, dw.ptr, 0.0, ws.ptr, ws.nbytes, st)
            rc = run()
            if rc:
                rows.append(f"{kind:5s} n{n} {hw}x{hw} {c:4d}->{k:4d} {r}x{r} s{s}  x{cnt}  UNSUPPORTED ({rc})")
                continue
            for _ in range(3):
                run()
            lib.nsk_event_record(e0, st)
            for _ in range(iters):
                run()
            lib.nsk_event_record(e1, st)
            lib.nsk_event_sync(e1)
            ms = C.c_float()
            lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
            us = 1000.0 * ms.value / iters
            tot = us * cnt
            grand += tot
            gflop += flops * cnt / 1e9
            rows.append(f"{kind:5s} n{n} {hw:3d}x{hw:<3d} {c:4d}->{k:4d} {r}x{r} s{s}  x{cnt}  {us:8.1f} us  "
                        f"{flops / us / 1e6:7.1f} TFLOP/s  total {tot:8.1f} us")
        del x, w, y, dw, ws
    for r_ in rows:
        print(r_)
    print(f"TOTAL conv time {grand:.1f} us for {gflop:.1f} GFLOP -> {gflop / grand * 1e3:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
