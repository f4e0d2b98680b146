"""New tape-recorded ops for CNN / GRU training (absent from the reference).

Each op follows the reference's recording pattern (autodiff.rec_* in
pkg/src/nsk/autodiff.py:165-248): compute the output with a libnskb kernel,
``record`` a node with its saved operands, and register a gradient rule.
Their CPU restatements (float64) live in oracle/restated.py.

Activations are NHWC bfloat16; parameters and their gradients float32 (the
tensor-core kernels read a bf16 shadow of each weight, refreshed by the
optimizer). Gradients always take the dtype of the tensor they belong to.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from . import _lib
from .side import SIDE
from ._lib import BF16, F32, ConvDesc, check
from .autodiff import SUNK, _internal_tensor, record, rule
from .errors import NskRuntimeError, NskTypeError
from .tensor import Buffer, Pool, Tensor, empty_tensor, release_tensor


class Workspace:
    """Grow-only scratch shared by kernels that need temporary device memory (stream-ordered reuse)."""

    def __init__(self):
        self.buf: Buffer | None = None
        self.retired: list[Buffer] = []  # outgrown buffers a side-stream kernel may still read (side.py)

    def get(self, nbytes: int) -> Buffer:
        if self.buf is None or self.buf.nbytes < nbytes:
            if self.buf is not None:
                self.retired.append(self.buf)
            self.buf = Buffer((max(nbytes, 1 << 20) + 3) // 4, F32)
        return self.buf


class _PerStream:
    """One Workspace per stream: kernels on the compute stream and on the side stream (forward branches,
    forked weight gradients) run concurrently and must never share scratch."""

    def __init__(self):
        self.ws: dict[int, Workspace] = {}

    def get(self, nbytes: int, stream: int | None = None) -> Buffer:
        st = _lib.stream() if stream is None else stream
        return self.ws.setdefault(st, Workspace()).get(nbytes)


BN_WS = _PerStream()
WGRAD_WS = _PerStream()  # split-K partials of conv weight gradients, keyed by the stream the wgrad runs on


def _temp_bf16(t: Tensor, pool: Pool) -> tuple[int, Tensor | None]:
    """bf16 pointer for ``t``: itself, a parameter's shadow, or a pooled cast copy (returned for release)."""
    if t.dtype == BF16:
        return t.ptr, None
    if t.param_name is not None:
        return t.bf16_ptr(), None
    tmp = empty_tensor(pool, t.shape, BF16)
    check(_lib.lib().nsk_cast(F32, t.ptr, BF16, tmp.ptr, t.numel, _lib.stream()))
    return tmp.ptr, tmp


# --- conv2d ---------------------------------------------------------------------------------

# Measurement hook (bench.py): an object with match(desc) / begin(stream) / end(stream) that brackets the matching
# conv fprop launches with CUDA events, so a kernel's duration is taken inside a real training step
KTIMER = None


def conv_out(h: int, k: int, stride: int, pad: int) -> int:
    return (h + 2 * pad - k) // stride + 1


def conv2d(x: Tensor, w: Tensor, stride: int, pad: int, pool: Pool, layout: str = "nhwc",
           bn_stats: bool = False) -> Tensor:
    """y[n,p,q,k] = sum_{r,s,c} x[n, p*st-pad+r, q*st-pad+s, c] * w[k,r,s,c]  (NHWC x KRSC -> NHWC, bf16).

    ``layout="nchw"`` accepts a host-layout float32 image batch [N, C, H, W] directly (image stems:
    the layout change is fused into the im2col gather; no input gradient). ``bn_stats`` (for a conv whose
    output goes straight into ``batchnorm``, see ``conv_bn``) makes the tcgen05 kernel also emit the BN
    channel statistics, so the BN needs no separate pass over y."""
    if x.rank != 4 or w.rank != 4:
        raise NskTypeError(f"conv2d needs NHWC input and KRSC filters, got {list(x.shape)} and {list(w.shape)}")
    nchw = layout == "nchw"
    if nchw:
        n, c, h, wd = x.shape
        if x.dtype != F32:
            raise NskTypeError("conv2d(layout='nchw') expects a float32 image batch")
    else:
        n, h, wd, c = x.shape
    k, r, s, c2 = w.shape
    if c != c2:
        raise NskTypeError(f"conv2d channel mismatch: input has {c}, filters expect {c2}")
    p, q = conv_out(h, r, stride, pad), conv_out(wd, s, stride, pad)
    if p < 1 or q < 1:
        raise NskTypeError(f"conv2d output would be empty for input {list(x.shape)}")
    desc = ConvDesc(n, h, wd, c, k, r, s, stride, pad, p, q)
    y = empty_tensor(pool, (n, p, q, k), BF16)
    lib = _lib.lib()
    st = _lib.stream()
    xp, xtmp = (x.ptr, None) if nchw else _temp_bf16(x, pool)
    wp = w.bf16_ptr() if w.dtype == F32 else w.ptr
    if c % 64 == 0 and not nchw:
        timer = KTIMER if KTIMER is not None and KTIMER.match(desc) else None
        if timer is not None:
            timer.begin(st)
        if bn_stats:
            # per-CTA channel partials for the BatchNorm consuming y (released by batchnorm)
            parts = empty_tensor(pool, (2 * _lib.ctx.sm_count, 2, k))
            nparts = C.c_int(0)
            check(lib.nsk_conv2d_fprop_stats(C.byref(desc), xp, wp, y.ptr, parts.ptr, parts.numel, C.byref(nparts),
                                             st))
            y.bn_partials = (parts, nparts.value)
        else:
            check(lib.nsk_conv2d_fprop(C.byref(desc), xp, wp, y.ptr, 0, st))
        if timer is not None:
            timer.end(st)
        saved = (x, w)
        attrs = {"desc": desc, "stem": False}
        if xtmp is not None:
            release_tensor(pool, xtmp)
    else:
        # small-channel stem: explicit im2col (K = R*S*C padded to a multiple of 8: TMA row pitch; the GEMM's
        # 64-wide K boxes read zeros past kp) + tcgen05 GEMM
        rsc = r * s * c
        kp = (rsc + 7) // 8 * 8
        cols = empty_tensor(pool, (n * p * q, kp), BF16)
        if nchw:
            check(lib.nsk_im2col_nchw(xp, cols.ptr, n, c, h, wd, r, s, stride, pad, p, q, kp, st))
        else:
            check(lib.nsk_im2col(xp, cols.ptr, n, h, wd, c, r, s, stride, pad, p, q, kp, st))
        if xtmp is not None:
            release_tensor(pool, xtmp)
        wpk = empty_tensor(pool, (k, kp), BF16)
        check(lib.nsk_fill_bf16(wpk.ptr, wpk.numel, 0.0, st))
        check(lib.nsk_memcpy2d_d2d(wpk.ptr, kp * 2, wp, rsc * 2, rsc * 2, k, st))
        check(lib.nsk_gemm(BF16, 0, 0, n * p * q, k, kp, cols.ptr, kp, wpk.ptr, kp, y.ptr, k, 0, None, 0.0, st))
        release_tensor(pool, wpk)
        _internal_tensor(cols)
        saved = (cols, w)
        attrs = {"desc": desc, "stem": True, "kp": kp, "nchw": nchw}
    record("conv2d", y, x, w, saved=saved, attrs=attrs)
    return y


@rule("conv2d")
def _r_conv2d(node, g, pool, sinks):
    desc = node.attrs["desc"]
    xin, w = node.saved
    lib = _lib.lib()
    st = _lib.stream()
    dx = dw = None
    gp, gtmp = _temp_bf16(g, pool)
    if node.inputs[0].requires_grad:
        acc = (node.acc_sinks or {}).get(0)
        xshape = tuple(node.inputs[0].tensor.shape)
        if acc is not None and (acc.dtype != BF16 or acc.shape != xshape or node.attrs["stem"]):
            acc = None
        dx = SUNK if acc is not None else empty_tensor(pool, xshape, BF16)
        wb = w.bf16_ptr() if w.dtype == F32 else w.ptr
        if node.attrs.get("nchw"):
            raise NskRuntimeError("conv2d(layout='nchw') input is image data and has no gradient")
        if node.attrs["stem"]:
            # dcols[M, Kp] = dy[M, K] . Wp[K, Kp] (Wp MN-major), then the col2im gather
            kp = node.attrs["kp"]
            rsc = desc.R * desc.S * desc.C
            m = desc.N * desc.P * desc.Q
            wpk = empty_tensor(pool, (desc.K, kp), BF16)
            check(lib.nsk_fill_bf16(wpk.ptr, wpk.numel, 0.0, st))
            check(lib.nsk_memcpy2d_d2d(wpk.ptr, kp * 2, wb, rsc * 2, rsc * 2, desc.K, st))
            dcols = empty_tensor(pool, (m, kp), F32)
            check(lib.nsk_gemm(BF16, 0, 1, m, kp, desc.K, gp, desc.K, wpk.ptr, kp, dcols.ptr, kp, 1, None, 0.0, st))
            check(lib.nsk_col2im(dcols.ptr, dx.ptr, desc.N, desc.H, desc.W, desc.C, desc.R, desc.S, desc.stride,
                                 desc.pad, desc.P, desc.Q, kp, st))
            release_tensor(pool, dcols)
            release_tensor(pool, wpk)
        elif _BNB_FUSE and (node.bnb_sinks or {}).get(0) is not None:
            # this dgrad completes the gradient of a BatchNorm(+ReLU) output: the epilogue stores it ReLU-masked
            # and emits the BatchNorm-backward channel sums, so _r_batchnorm skips its reduction pass
            bn = node.bnb_sinks[0]
            target = acc if acc is not None else dx
            mask = bn.saved[4] if bn.attrs["relu"] else None
            parts = empty_tensor(pool, (2 * _lib.ctx.sm_count, 2, desc.C))
            nparts = C.c_int(0)
            check(lib.nsk_conv2d_dgrad_bnstats(C.byref(desc), gp, wb, target.ptr, 1.0 if acc is not None else 0.0,
                                               bn.saved[0].ptr, None if mask is None else mask.ptr, parts.ptr,
                                               parts.numel, C.byref(nparts), st))
            if nparts.value > 0:
                target.bnb_partials = (parts, nparts.value)
            else:  # tile configuration without room for the statistics: plain dgrad ran, BN reduces itself
                release_tensor(pool, parts)
        elif acc is not None:  # second contribution: accumulate into the pending gradient in the epilogue
            check(lib.nsk_conv2d_dgrad_acc(C.byref(desc), gp, wb, acc.ptr, 1.0, st))
        else:
            check(lib.nsk_conv2d_dgrad(C.byref(desc), gp, wb, dx.ptr, st))
    if node.inputs[1].requires_grad:
        if sinks[1] is not None:
            out_ptr, beta, dw = sinks[1].ptr, 1.0, SUNK
        else:
            dwt = empty_tensor(pool, w.shape, F32)
            out_ptr, beta, dw = dwt.ptr, 0.0, dwt
        if node.attrs["stem"]:
            # dW[k, rsc] = dy^T . cols : A = dy [M][K] (MN-major), B = cols [M][Kp] (MN-major), N = R*S*C
            m = desc.N * desc.P * desc.Q
            rsc = desc.R * desc.S * desc.C
            check(lib.nsk_gemm(BF16, 1, 1, desc.K, rsc, m, gp, desc.K, xin.ptr, node.attrs["kp"], out_ptr, rsc, 1,
                               None, beta, st))
        else:
            xp, xtmp = _temp_bf16(xin, pool)
            need = lib.nsk_conv2d_wgrad_workspace(C.byref(desc))
            wst = st
            if sinks[1] is not None and SIDE.enabled():
                # overlap the weight gradient with the rest of backward (side.py); its inputs stay alive to the join
                wst = SIDE.fork(xin.buffer, g.buffer, None if xtmp is None else xtmp.buffer,
                                None if gtmp is None else gtmp.buffer)
            ws = WGRAD_WS.get(need, wst)
            check(lib.nsk_conv2d_wgrad(C.byref(desc), xp, gp, out_ptr, beta, ws.ptr, ws.nbytes, wst))
            if xtmp is not None:
                release_tensor(pool, xtmp)
    if gtmp is not None:
        release_tensor(pool, gtmp)
    return [dx, dw]


# BatchNorm backward statistics fused into the dgrad that completes the BatchNorm output's gradient
# (nsk_conv2d_dgrad_bnstats). Off by default: measured on B200 the statistics epilogue lengthens the
# latency-bound epilogue of the weight-resident 64-channel dgrad by more than the separate reduction pass costs
# (2.08 -> 2.13 ms/step); NSK_BNB_FUSE=1 enables it (tests/test_gpu_parity_c2.py checks it either way)
_BNB_FUSE = os.environ.get("NSK_BNB_FUSE", "0") == "1"


# --- batchnorm (+ residual, + relu) ---------------------------------------------------------------

def conv_bn(x: Tensor, w: Tensor, gb: Tensor, stride: int, pad: int, pool: Pool, relu: bool = False,
            residual: Tensor | None = None, layout: str = "nhwc", training: bool = True) -> Tensor:
    """conv2d followed by batchnorm (two recorded ops, same gradients); in training the conv kernel emits the
    BN channel statistics so the normalisation reads its input once."""
    return batchnorm(conv2d(x, w, stride, pad, pool, layout=layout, bn_stats=training), gb, pool, relu=relu,
                     residual=residual, training=training)


_RUNNING: "weakref.WeakKeyDictionary[Tensor, Buffer]" = weakref.WeakKeyDictionary()
BN_MOMENTUM = 0.1


def bn_running(gb: Tensor) -> Buffer:
    """The running statistics [2, C] (mean row, unbiased variance row) of a BatchNorm parameter, created on
    first use as (0, 1); training forwards update them with momentum BN_MOMENTUM, eval forwards read them."""
    buf = _RUNNING.get(gb)
    if buf is None:
        c = gb.shape[1]
        buf = Buffer(2 * c, F32)
        buf.upload(np.concatenate([np.zeros(c, np.float32), np.ones(c, np.float32)]))
        _RUNNING[gb] = buf
    return buf


def batchnorm(x: Tensor, gb: Tensor, pool: Pool, relu: bool = False, residual: Tensor | None = None,
              eps: float = 1e-5, training: bool = True) -> Tensor:
    """Batch norm over N*H*W per channel, gamma_beta = [2, C]; optional residual add and ReLU. Training mode
    normalises with the batch statistics (and updates the running ones); eval mode (``training=False``)
    with the running statistics and records nothing for backward."""
    if x.dtype != BF16:
        raise NskTypeError("batchnorm expects a bf16 NHWC activation")
    c = x.shape[-1]
    if gb.shape != (2, c):
        raise NskTypeError(f"batchnorm parameters must be [2, {c}], got {list(gb.shape)}")
    if residual is not None and (residual.shape != x.shape or residual.dtype != BF16):
        raise NskTypeError("batchnorm residual must match the input shape (bf16)")
    rows = x.numel // c
    lib = _lib.lib()
    st = _lib.stream()
    y = empty_tensor(pool, x.shape, BF16)
    running = bn_running(gb)
    if not training:
        ws = BN_WS.get(lib.nsk_bn_workspace(rows, c))
        check(lib.nsk_bn_fwd_eval(x.ptr, gb.ptr, running.ptr, y.ptr, rows, c, float(eps), int(relu),
                                  None if residual is None else residual.ptr, ws.ptr, st))
        if x.bn_partials is not None:
            release_tensor(pool, x.bn_partials[0])
            x.bn_partials = None
        return y
    mean = _internal_tensor(empty_tensor(pool, (c,)))
    invstd = _internal_tensor(empty_tensor(pool, (c,)))
    ws = BN_WS.get(lib.nsk_bn_workspace(rows, c))
    # ReLU mask for the backward: one bit per element (rows*C/8 bytes, held in a float32 buffer)
    mask = _internal_tensor(empty_tensor(pool, ((x.numel // 8 + 3) // 4,))) if relu else None
    mp = None if mask is None else mask.ptr
    rp = None if residual is None else residual.ptr
    parts = x.bn_partials
    if parts is not None:
        check(lib.nsk_bn_fwd_partials(parts[0].ptr, parts[1], x.ptr, gb.ptr, y.ptr, mean.ptr, invstd.ptr, rows, c,
                                      float(eps), int(relu), rp, mp, running.ptr, float(BN_MOMENTUM), ws.ptr, st))
        release_tensor(pool, parts[0])
        x.bn_partials = None
    else:
        check(lib.nsk_bn_fwd(x.ptr, gb.ptr, y.ptr, mean.ptr, invstd.ptr, rows, c, float(eps), int(relu), rp, mp,
                             running.ptr, float(BN_MOMENTUM), ws.ptr, st))
    saved = (x, gb, mean, invstd) + ((mask,) if relu else ())
    record("batchnorm", y, x, gb, residual, saved=saved, attrs={"relu": relu, "rows": rows, "c": c})
    return y


@rule("batchnorm")
def _r_batchnorm(node, g, pool, sinks):
    x, gb, mean, invstd = node.saved[:4]
    mask = node.saved[4] if node.attrs["relu"] else None
    rows, c = node.attrs["rows"], node.attrs["c"]
    lib = _lib.lib()
    st = _lib.stream()
    if g.dtype != BF16:
        raise NskRuntimeError("batchnorm gradient must be bf16")
    dx = empty_tensor(pool, x.shape, BF16) if node.inputs[0].requires_grad else None
    res_node = node.inputs[2]
    dres = empty_tensor(pool, x.shape, BF16) if (res_node is not None and res_node.requires_grad) else None
    if sinks[1] is not None:
        dgb_ptr, beta, dgb = sinks[1].ptr, 1.0, SUNK
    else:
        t = empty_tensor(pool, (2, c))
        dgb_ptr, beta, dgb = t.ptr, 0.0, t
    scratch_dx = None
    if dx is None:
        scratch_dx = empty_tensor(pool, x.shape, BF16)
    ws = BN_WS.get(lib.nsk_bn_workspace(rows, c))
    parts = g.bnb_partials
    if parts is not None:  # g arrives ReLU-masked with its channel sums (the dgrad that completed it)
        g.bnb_partials = None
        check(lib.nsk_bn_bwd_partials(parts[0].ptr, parts[1], g.ptr, x.ptr, gb.ptr, mean.ptr, invstd.ptr,
                                      (dx or scratch_dx).ptr, None if dres is None else dres.ptr, dgb_ptr, beta,
                                      rows, c, ws.ptr, st))
        release_tensor(pool, parts[0])
    else:
        check(lib.nsk_bn_bwd(g.ptr, x.ptr, None if mask is None else mask.ptr, gb.ptr, mean.ptr, invstd.ptr,
                             (dx or scratch_dx).ptr, None if dres is None else dres.ptr, dgb_ptr, beta, rows, c,
                             ws.ptr, st))
    if scratch_dx is not None:
        release_tensor(pool, scratch_dx)
    if not node.inputs[1].requires_grad:
        if dgb is not SUNK and dgb is not None:
            release_tensor(pool, dgb)
        dgb = None
    return [dx, dgb, dres]


# --- pooling / reshape / layout -------------------------------------------------------------------

def avgpool_global(x: Tensor, pool: Pool) -> Tensor:
    """[N, H, W, C] -> [N, C] float32 mean over H*W."""
    n, h, w, c = x.shape
    y = empty_tensor(pool, (n, c))
    check(_lib.lib().nsk_avgpool_fwd(x.dtype, x.ptr, y.ptr, n, h * w, c, _lib.stream()))
    record("avgpool", y, x, attrs={"shape": x.shape, "dtype": x.dtype})
    return y


@rule("avgpool")
def _r_avgpool(node, g, pool, sinks):
    shape, dtype = node.attrs["shape"], node.attrs["dtype"]
    n, h, w, c = shape
    dx = empty_tensor(pool, shape, dtype)
    check(_lib.lib().nsk_avgpool_bwd(g.ptr, dtype, dx.ptr, n, h * w, c, _lib.stream()))
    return [dx]


def maxpool(x: Tensor, k: int, stride: int, pad: int, pool: Pool) -> Tensor:
    """k x k max-pool (NHWC bf16); the first-maximum window position is kept as one byte per output for the
    backward (restated.maxpool_bwd tie rule)."""
    if x.dtype != BF16:
        raise NskTypeError("maxpool expects a bf16 NHWC activation")
    n, h, w, c = x.shape
    p, q = conv_out(h, k, stride, pad), conv_out(w, k, stride, pad)
    y = empty_tensor(pool, (n, p, q, c), BF16)
    arg = _internal_tensor(empty_tensor(pool, ((n * p * q * c + 3) // 4,)))  # bytes in a float32 buffer
    check(_lib.lib().nsk_maxpool_fwd(x.ptr, y.ptr, arg.ptr, n, h, w, c, k, stride, pad, p, q, _lib.stream()))
    record("maxpool", y, x, saved=(arg,), attrs={"k": k, "stride": stride, "pad": pad, "shape": x.shape})
    return y


@rule("maxpool")
def _r_maxpool(node, g, pool, sinks):
    (arg,) = node.saved
    a = node.attrs
    n, h, w, c = a["shape"]
    _, p, q, _ = g.shape
    dx = empty_tensor(pool, a["shape"], BF16)
    check(_lib.lib().nsk_maxpool_bwd(arg.ptr, g.ptr, dx.ptr, n, h, w, c, a["k"], a["stride"], a["pad"], p, q,
                                     _lib.stream()))
    return [dx]


def reshape(x: Tensor, shape, pool: Pool) -> Tensor:
    """A recorded copy with a new shape (row-major order kept; NHWC flatten)."""
    shape = tuple(int(d) for d in shape)
    if int(np.prod(shape)) != x.numel:
        raise NskTypeError(f"cannot reshape {list(x.shape)} to {list(shape)}")
    y = empty_tensor(pool, shape, x.dtype)
    check(_lib.lib().nsk_memcpy_d2d(y.ptr, x.ptr, x.buffer.nbytes, _lib.stream()))
    record("reshape", y, x, attrs={"shape": x.shape})
    return y


@rule("reshape")
def _r_reshape(node, g, pool, sinks):
    dx = empty_tensor(pool, node.attrs["shape"], g.dtype)
    check(_lib.lib().nsk_memcpy_d2d(dx.ptr, g.ptr, g.buffer.nbytes, _lib.stream()))
    return [dx]


def cast(x: Tensor, dtype: int, pool: Pool) -> Tensor:
    if x.dtype == dtype:
        return x
    y = empty_tensor(pool, x.shape, dtype)
    check(_lib.lib().nsk_cast(x.dtype, x.ptr, dtype, y.ptr, x.numel, _lib.stream()))
    record("cast", y, x, attrs={"dtype": x.dtype})
    return y


@rule("cast")
def _r_cast(node, g, pool, sinks):
    dt = node.attrs["dtype"]
    dx = empty_tensor(pool, g.shape, dt)
    check(_lib.lib().nsk_cast(g.dtype, g.ptr, dt, dx.ptr, g.numel, _lib.stream()))
    return [dx]


def nchw_to_nhwc(x: Tensor, pool: Pool, channels_pad: int | None = None) -> Tensor:
    """Host-layout images [N, C, H, W] float32 -> NHWC bf16 (no gradient: data preparation)."""
    n, c, h, w = x.shape
    cp = channels_pad or c
    y = empty_tensor(pool, (n, h, w, cp), BF16)
    check(_lib.lib().nsk_nchw_to_nhwc(x.ptr, y.ptr, n, c, h, w, cp, _lib.stream()))
    record("layout", y, x)
    return y


@rule("layout")
def _r_layout(node, g, pool, sinks):
    raise NskRuntimeError("nchw_to_nhwc is a data-preparation op and has no gradient")


# --- sequence ops: embedding + fused GRU -------------------------------------------------------------

def embedding(tokens: Tensor, table: Tensor, pool: Pool, dtype: int = F32) -> Tensor:
    """tokens [B, T] (float ids, as loaded) -> rows of table [V, E], time-major [T*B, E] (float32, or bf16 when
    the consumer is a bf16 tensor-core GEMM: the GRU input projection).

    Equals onehot(tokens) @ E exactly (a one-term float64 sum), the reference's embedding path
    (tensor.py:299-317 + :213-229), rounded to the output dtype; range errors keep onehot's message."""
    from .tensor import check_index_values, device_index_check

    if tokens.rank != 2 or table.rank != 2:
        raise NskTypeError(f"embedding needs [B, T] tokens and a [V, E] table, got {list(tokens.shape)}, "
                           f"{list(table.shape)}")
    b, t = tokens.shape
    v, e = table.shape
    if tokens.host_src is not None:
        check_index_values(tokens.host_src, v, "onehot")
    else:
        device_index_check(Tensor((b * t,), tokens.buffer), v, "onehot")
    out = empty_tensor(pool, (t * b, e), dtype)
    check(_lib.lib().nsk_embedding_fwd(table.ptr, tokens.ptr, b * t, e, v, t, dtype, out.ptr, None, _lib.stream()))
    record("embedding", out, tokens, table, saved=(tokens,), attrs={"T": t, "V": v})
    return out


@rule("embedding")
def _r_embedding(node, g, pool, sinks):
    (tokens,) = node.saved
    v, e = node.inputs[1].tensor.shape
    if sinks[1] is not None:
        out_ptr, dt = sinks[1].ptr, SUNK  # scatter-add straight into the cached gradient
    else:
        dt = empty_tensor(pool, (v, e), F32)
        dt.buffer.fill(0.0)
        out_ptr = dt.ptr
    check(_lib.lib().nsk_embedding_bwd(g.ptr, g.dtype, tokens.ptr, tokens.numel, e, node.attrs["T"], out_ptr,
                                       _lib.stream()))
    return [None, dt]


GRU_WS = Workspace()


def gru(x: Tensor, w: Tensor, b: Tensor, u: Tensor, c: Tensor, steps: int, pool: Pool) -> Tensor:
    """Fused GRU over a time-major input x [T*B, E] -> final hidden state h_T [B, H] (h_0 = 0).

    w [3H, E], b [3H], u [3H, H], c [3H] stack the (r, z, n) gates. Same function as the reference
    composition r = s(x W_r^T + b_r + h U_r^T + c_r), z likewise, n = tanh(x W_n^T + b_n + r (h U_n^T + c_n)),
    h' = n - z n + z h; input projections for all steps are one tcgen05 GEMM."""
    from .tensor import _gemm

    tb, e = x.shape
    h3, e2 = w.shape
    h = h3 // 3
    if e2 != e or h3 % 3 or u.shape != (h3, h) or b.shape != (h3,) or c.shape != (h3,) or tb % steps:
        raise NskTypeError("gru: inconsistent shapes")
    bsz = tb // steps
    lib, st = _lib.lib(), _lib.stream()
    gx = empty_tensor(pool, (tb, h3), F32)
    if x.dtype == BF16:  # bf16 tensor-core input projection (W through its bf16 shadow), fp32 out + b
        _gemm(x.ptr, 0, e, w.bf16_ptr(), 0, e, tb, h3, e, gx.ptr, h3, dtype=BF16, bias_ptr=b.ptr)
    else:
        _gemm(x.ptr, 0, e, w.ptr, 0, e, tb, h3, e, gx.ptr, h3, dtype=F32, bias_ptr=b.ptr)
    hs = _internal_tensor(empty_tensor(pool, ((steps + 1) * bsz, h), F32))
    check(lib.nsk_fill_f32(hs.ptr, bsz * h, 0.0, st))
    gates = _internal_tensor(empty_tensor(pool, (tb, 4 * h), F32))
    tc = _gru_tc(bsz, h)
    hsb = None
    if tc:  # tensor-core recurrence: one cluster, U resident as bf16 (gru_tc.cu); also a bf16 copy of h for dU
        hsb = _internal_tensor(empty_tensor(pool, ((steps + 1) * bsz, h), BF16))
        ws = GRU_WS.get(lib.nsk_gru_tc_workspace(bsz, h))
        check(lib.nsk_gru_fwd_tc(gx.ptr, u.bf16_ptr(), c.ptr, steps, bsz, h, hs.ptr, hsb.ptr, gates.ptr, ws.ptr,
                                 ws.nbytes, st))
    else:  # shapes the cluster kernel does not tile: fp32 cooperative kernel (gru.cu)
        check(lib.nsk_gru_fwd(gx.ptr, u.ptr, c.ptr, steps, bsz, h, hs.ptr, gates.ptr, st))
    release_tensor(pool, gx)
    out = empty_tensor(pool, (bsz, h), F32)
    check(lib.nsk_memcpy_d2d(out.ptr, hs.ptr + 4 * steps * bsz * h, 4 * bsz * h, st))
    saved = (x, hs, gates, w, u) + ((hsb,) if tc else ())
    record("gru", out, x, w, b, u, c, saved=saved, attrs={"T": steps, "B": bsz, "H": h, "E": e, "tc": tc})
    return out


def _gru_tc(bsz: int, h: int) -> bool:
    """The tcgen05 cluster recurrence covers 1 <= B <= 64, H in 128..512 (H % 64 == 0); NSK_GRU_TC=0 forces the
    fp32 cooperative kernel (A/B and precision studies)."""
    return os.environ.get("NSK_GRU_TC", "1") != "0" and bool(_lib.lib().nsk_gru_tc_supported(bsz, h))


@rule("gru")
def _r_gru(node, g, pool, sinks):
    from .tensor import _gemm, _Operands

    tc = node.attrs.get("tc")
    x, hs, gates, w, u = node.saved[:5]
    T, B, H, E = (node.attrs[k] for k in ("T", "B", "H", "E"))
    H3, TB = 3 * H, T * B
    lib, st = _lib.lib(), _lib.stream()
    outs = [None] * 5

    def target(i, shape):
        if sinks[i] is not None:
            return sinks[i].ptr, 1.0, SUNK
        t = empty_tensor(pool, shape, F32)
        return t.ptr, 0.0, t

    dhs = empty_tensor(pool, (TB, H), F32)
    check(lib.nsk_fill_f32(dhs.ptr, (T - 1) * B * H, 0.0, st))
    check(lib.nsk_memcpy_d2d(dhs.ptr + 4 * (T - 1) * B * H, g.ptr, 4 * B * H, st))
    dh0 = empty_tensor(pool, (B, H), F32)
    if tc:
        # the cluster kernel emits dgx / dgh as bf16 GEMM operands and reduces the bias gradients itself
        hsb = node.saved[5]
        dgx = empty_tensor(pool, (TB, H3), BF16)
        dgh = empty_tensor(pool, (TB, H3), BF16)
        scratch = []
        bias = []
        for i in (2, 4):
            if node.inputs[i].requires_grad:
                ptr, beta, outs[i] = target(i, (H3,))
            else:
                tmp = empty_tensor(pool, (H3,), F32)
                scratch.append(tmp)
                ptr, beta = tmp.ptr, 0.0
            bias.append((ptr, beta))
        ws = GRU_WS.get(lib.nsk_gru_tc_workspace(B, H))
        check(lib.nsk_gru_bwd_tc(dhs.ptr, u.bf16_ptr(), hs.ptr, gates.ptr, T, B, H, dgx.ptr, dgh.ptr, dh0.ptr,
                                 bias[0][0], bias[0][1], bias[1][0], bias[1][1], ws.ptr, ws.nbytes, st))
        for tmp in scratch:
            release_tensor(pool, tmp)
        hprev = Tensor((TB, H), Buffer(TB * H, BF16, base=hsb.buffer, offset=0))
    else:
        dgx = empty_tensor(pool, (TB, H3), F32)
        dgh = empty_tensor(pool, (TB, H3), F32)
        ws = GRU_WS.get(lib.nsk_gru_bwd_workspace(T, B, H))
        check(lib.nsk_gru_bwd(dhs.ptr, u.ptr, hs.ptr, gates.ptr, T, B, H, dgx.ptr, dgh.ptr, dh0.ptr, ws.ptr,
                              ws.nbytes, st))
        hprev = Tensor((TB, H), Buffer(TB * H, F32, base=hs.buffer, offset=0))
    release_tensor(pool, dhs)
    release_tensor(pool, dh0)

    # bf16 operands, fp32 accumulation for the batched weight / input gradients (K = T*B steps)
    with _Operands(pool, BF16, dgx, dgh, x, w, hprev) as (pgx, pgh, px, pw, ph):
        if node.inputs[0].requires_grad:
            xdt = node.inputs[0].tensor.dtype  # the gradient takes the input's dtype
            dx = empty_tensor(pool, (TB, E), xdt)
            _gemm(pgx, 0, H3, pw, 1, E, TB, E, H3, dx.ptr, E, dtype=BF16, out_f32=xdt == F32)  # dx = dgx . W
            outs[0] = dx
        if node.inputs[1].requires_grad:
            ptr, beta, outs[1] = target(1, (H3, E))
            _gemm(pgx, 1, H3, px, 1, E, H3, E, TB, ptr, E, dtype=BF16, beta=beta)  # dW = dgx^T . x
        if node.inputs[3].requires_grad:
            ptr, beta, outs[3] = target(3, (H3, H))
            _gemm(pgh, 1, H3, ph, 1, H, H3, H, TB, ptr, H, dtype=BF16, beta=beta)  # dU = dgh^T . h_{t-1}
    if not tc:
        if node.inputs[2].requires_grad:
            ptr, beta, outs[2] = target(2, (H3,))
            check(lib.nsk_colsum(F32, dgx.ptr, ptr, TB, H3, beta, st))
        if node.inputs[4].requires_grad:
            ptr, beta, outs[4] = target(4, (H3,))
            check(lib.nsk_colsum(F32, dgh.ptr, ptr, TB, H3, beta, st))
    release_tensor(pool, dgx)
    release_tensor(pool, dgh)
    return outs
