"""Compare split-K conv passes against the unsplit kernels (NSK_CONV_SPLIT toggled per call): fprop (+ BN
statistics partials folded over parts) and dgrad, several small-M shapes. Prints max normwise differences."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200._lib import BF16, F32, ConvDesc  # noqa: E402
from paper_2409_11600_b200.tensor import Buffer  # noqa: E402

_lib.ctx.init(0)
lib, st = _lib.lib(), _lib.stream()
rng = np.random.default_rng(0)


def bf(a):
    return (a.astype(np.float32).view(np.uint32) + 0x8000 & 0xFFFF0000).view(np.float32)


for (n, hw, c, k, r, s, pad) in [(16, 4, 512, 512, 3, 1, 1), (16, 8, 256, 512, 3, 2, 1), (16, 8, 256, 256, 3, 1, 1),
                                 (64, 4, 512, 512, 3, 1, 1), (256, 4, 512, 512, 3, 1, 1)]:
    p = (hw + 2 * pad - r) // s + 1
    d = ConvDesc(n, hw, hw, c, k, r, r, s, pad, p, p)
    x = Buffer(n * hw * hw * c, BF16); x.upload(bf(rng.standard_normal(n * hw * hw * c)))
    w = Buffer(k * r * r * c, BF16); w.upload(bf(rng.standard_normal(k * r * r * c) / np.sqrt(r * r * c)))
    y = Buffer(n * p * p * k, BF16)
    nst = int(lib.nsk_conv2d_stats_floats(k)) if hasattr(lib, "nsk_conv2d_stats_floats") else 2 * 148 * 2 * k * 2
    parts = Buffer(nst, F32)
    res = {}
    for sp in ("0", "1"):
        os.environ["NSK_CONV_SPLIT"] = sp
        npart = C.c_int(0)
        _lib.check(lib.nsk_conv2d_fprop_stats(C.byref(d), x.ptr, w.ptr, y.ptr, parts.ptr, nst, C.byref(npart), st))
        _lib.sync()
        pr = parts.host()[: npart.value * 2 * k].reshape(npart.value, 2, k).astype(np.float64).sum(0)
        res[sp] = (y.host().copy(), pr)
    dy = y
    dx = Buffer(n * hw * hw * c, BF16)
    dres = {}
    if s == 1:
        for sp in ("0", "1"):
            os.environ["NSK_CONV_SPLIT"] = sp
            _lib.check(lib.nsk_conv2d_dgrad(C.byref(d), dy.ptr, w.ptr, dx.ptr, st))
            _lib.sync()
            dres[sp] = dx.host().copy()
    a, b = res["0"][0].astype(np.float64), res["1"][0].astype(np.float64)
    e_y = np.linalg.norm(a - b) / np.linalg.norm(a)
    e_s = np.abs(res["0"][1] - res["1"][1]).max() / np.abs(res["0"][1]).max()
    e_dx = (np.linalg.norm(dres["0"].astype(np.float64) - dres["1"]) / np.linalg.norm(dres["0"])) if dres else -1
    print(f"n{n} {hw}x{hw} {c}->{k} s{s}: y {e_y:.2e} stats {e_s:.2e} dx {e_dx:.2e}  |y| {np.abs(a).mean():.3g} "
          f"{np.abs(b).mean():.3g}  npart {npart.value}")
