"""Early GPU probe of the tcgen05 GEMM / conv kernels (torch used only as plumbing + reference)."""
import ctypes
import os
import sys
import time

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2409_11600_b200", "libnskb.so"))
lib.nsk_last_error.restype = ctypes.c_char_p
lib.nsk_conv2d_wgrad_workspace.restype = ctypes.c_uint64


class Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("N", "H", "W", "C", "K", "R", "S", "stride", "pad", "P", "Q")]


def chk(rc):
    if rc != 0:
        raise RuntimeError(lib.nsk_last_error().decode())


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def rel(a, b):
    return ((a.double() - b.double()).norm() / (b.double().norm() + 1e-30)).item()


def gemm_case(dtype, a_mn, b_mn, M, N, K):
    dt = torch.bfloat16 if dtype == 1 else torch.float32
    A = torch.randn(M, K, device="cuda").to(dt)
    B = torch.randn(N, K, device="cuda").to(dt)
    Ast = A.t().contiguous() if a_mn else A
    Bst = B.t().contiguous() if b_mn else B
    lda = M if a_mn else K
    ldb = N if b_mn else K
    C = torch.full((M, N), float("nan"), device="cuda")
    bias = torch.randn(N, device="cuda")
    chk(lib.nsk_gemm(dtype, a_mn, b_mn, M, N, K, P(Ast), ctypes.c_longlong(lda), P(Bst), ctypes.c_longlong(ldb),
                     P(C), ctypes.c_longlong(N), 1, P(bias), ctypes.c_float(0.0), stream()))
    torch.cuda.synchronize()
    if dtype == 0:
        Ar = A.view(torch.int32).bitwise_and(-8192).view(torch.float32)  # truncate to tf32-ish for the reference
        Br = B.view(torch.int32).bitwise_and(-8192).view(torch.float32)
        ref = A.double() @ B.double().t() + bias.double()
        e = rel(C, ref)
    else:
        ref = A.double() @ B.double().t() + bias.double()
        e = rel(C, ref)
    print(f"gemm dt={dtype} a_mn={a_mn} b_mn={b_mn} M={M} N={N} K={K}: rel={e:.2e}", flush=True)
    return e


def conv_case(N, H, W, C, K, R, stride, pad):
    Pp = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - R) // stride + 1
    d = Desc(N, H, W, C, K, R, R, stride, pad, Pp, Q)
    x = torch.randn(N, H, W, C, device="cuda").bfloat16()
    w = (torch.randn(K, R, R, C, device="cuda") / (C * R * R) ** 0.5).bfloat16()
    y = torch.full((N, Pp, Q, K), float("nan"), device="cuda").bfloat16()
    print("  fprop...", flush=True)
    chk(lib.nsk_conv2d_fprop(ctypes.byref(d), P(x), P(w), P(y), 0, stream()))
    torch.cuda.synchronize()
    xr = x.float().permute(0, 3, 1, 2)
    wr = w.float().permute(0, 3, 1, 2)
    ref = F.conv2d(xr.double(), wr.double(), stride=stride, padding=pad).permute(0, 2, 3, 1)
    e1 = rel(y.float(), ref)
    # dgrad
    dy = torch.randn(N, Pp, Q, K, device="cuda").bfloat16()
    dx = torch.full((N, H, W, C), float("nan"), device="cuda").bfloat16()
    print("  dgrad...", flush=True)
    chk(lib.nsk_conv2d_dgrad(ctypes.byref(d), P(dy), P(w), P(dx), stream()))
    torch.cuda.synchronize()
    dyr = dy.double().permute(0, 3, 1, 2)
    refdx = torch.nn.grad.conv2d_input((N, C, H, W), wr.double(), dyr, stride=stride, padding=pad).permute(0, 2, 3, 1)
    e2 = rel(dx.float(), refdx)
    # wgrad
    wsb = lib.nsk_conv2d_wgrad_workspace(ctypes.byref(d))
    ws = torch.empty(wsb // 4 + 1, device="cuda")
    dw = torch.full((K, R, R, C), float("nan"), device="cuda")
    print("  wgrad...", flush=True)
    chk(lib.nsk_conv2d_wgrad(ctypes.byref(d), P(x), P(dy), P(dw), ctypes.c_float(0.0), P(ws), ctypes.c_uint64(wsb),
                             stream()))
    torch.cuda.synchronize()
    refdw = torch.nn.grad.conv2d_weight(xr.double(), (K, C, R, R), dyr, stride=stride, padding=pad).permute(0, 2, 3, 1)
    e3 = rel(dw, refdw)
    print(f"conv N={N} H={H} C={C} K={K} R={R} s={stride} p={pad}: fprop {e1:.2e} dgrad {e2:.2e} wgrad {e3:.2e}",
          flush=True)
    return max(e1, e2, e3)


def bench_conv(N, H, W, C, K, R, stride, pad, iters=20):
    Pp = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - R) // stride + 1
    d = Desc(N, H, W, C, K, R, R, stride, pad, Pp, Q)
    x = torch.randn(N, H, W, C, device="cuda").bfloat16()
    w = torch.randn(K, R, R, C, device="cuda").bfloat16()
    y = torch.empty(N, Pp, Q, K, device="cuda").bfloat16()
    dy = torch.randn(N, Pp, Q, K, device="cuda").bfloat16()
    dx = torch.empty(N, H, W, C, device="cuda").bfloat16()
    wsb = lib.nsk_conv2d_wgrad_workspace(ctypes.byref(d))
    ws = torch.empty(wsb // 4 + 1, device="cuda")
    dw = torch.empty(K, R, R, C, device="cuda")
    flops = 2.0 * N * Pp * Q * K * C * R * R
    res = {}
    for name, fn in (
        ("fprop", lambda: lib.nsk_conv2d_fprop(ctypes.byref(d), P(x), P(w), P(y), 0, stream())),
        ("dgrad", lambda: lib.nsk_conv2d_dgrad(ctypes.byref(d), P(dy), P(w), P(dx), stream())),
        ("wgrad", lambda: lib.nsk_conv2d_wgrad(ctypes.byref(d), P(x), P(dy), P(dw), ctypes.c_float(0.0), P(ws),
                                               ctypes.c_uint64(wsb), stream())),
    ):
        for _ in range(3):
            chk(fn())
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        res[name] = (ms, flops / ms / 1e9)
    print(f"bench conv N={N} H={H} C={C} K={K} R={R} s={stride}: " +
          " ".join(f"{k} {v[0]*1000:.1f}us {v[1]:.0f}TF" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    torch.manual_seed(0)
    errs = []
    for case in [(1, 0, 0, 256, 128, 256), (1, 0, 0, 300, 200, 320), (1, 1, 0, 256, 128, 192), (1, 0, 1, 256, 128, 192),
                 (1, 1, 1, 384, 256, 128), (0, 0, 0, 256, 64, 128), (0, 1, 1, 256, 64, 96), (1, 0, 0, 256, 10, 512)]:
        errs.append(gemm_case(*case))
    for case in [(2, 32, 32, 64, 64, 3, 1, 1), (2, 32, 32, 64, 128, 3, 2, 1), (2, 32, 32, 64, 128, 1, 2, 0),
                 (4, 16, 16, 128, 128, 3, 1, 1), (8, 8, 8, 256, 256, 3, 1, 1), (16, 4, 4, 512, 512, 3, 1, 1),
                 (16, 8, 8, 256, 512, 3, 2, 1)]:
        errs.append(conv_case(*case))
    print("MAXERR", max(errs))
    if "--bench" in sys.argv:
        for case in [(256, 32, 32, 64, 64, 3, 1, 1), (256, 16, 16, 128, 128, 3, 1, 1), (256, 8, 8, 256, 256, 3, 1, 1),
                     (256, 4, 4, 512, 512, 3, 1, 1), (256, 32, 32, 64, 128, 3, 2, 1)]:
            bench_conv(*case)
