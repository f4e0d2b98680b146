"""ctypes binding of libnskb.so (include/nskb.h) and the device context.

There is no fallback: if the shared library is missing or no CUDA device is
present, every op raises. ``check`` maps the ABI status codes onto the
reference's error types (include/nskb.h header comment).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NskRuntimeError, NskTypeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NSK_LIB") or os.path.join(_HERE, "libnskb.so")  # NSK_LIB: A/B builds (tools/)

F32, BF16 = 0, 1
DTYPE_SIZE = {F32: 4, BF16: 2}
DTYPE_NAME = {F32: "f32", BF16: "bf16"}

vp, i32, u64, i64, f32, f64 = C.c_void_p, C.c_int, C.c_uint64, C.c_longlong, C.c_float, C.c_double


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "H", "W", "C", "K", "R", "S", "stride", "pad", "P", "Q")]


# name -> (restype, argtypes); mirrors include/nskb.h
SIGNATURES = {
    "nsk_last_error": (C.c_char_p, []),
    "nsk_abi_version": (i32, []),
    "nsk_init": (i32, [i32]),
    "nsk_device_info": (i32, [C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(u64)]),
    "nsk_arena_alloc": (i32, [u64, vp, C.POINTER(vp)]),
    "nsk_arena_free": (i32, [vp, vp]),
    "nsk_arena_stats": (i32, [C.POINTER(u64)]),
    "nsk_arena_trim": (i32, []),
    "nsk_pinned_alloc": (i32, [u64, C.POINTER(vp)]),
    "nsk_pinned_free": (i32, [vp]),
    "nsk_memcpy_h2d": (i32, [vp, vp, u64, vp]),
    "nsk_memcpy_d2h": (i32, [vp, vp, u64, vp]),
    "nsk_memcpy_d2d": (i32, [vp, vp, u64, vp]),
    "nsk_memcpy2d_d2d": (i32, [vp, u64, vp, u64, u64, u64, vp]),
    "nsk_stream_create": (i32, [C.POINTER(vp)]),
    "nsk_stream_destroy": (i32, [vp]),
    "nsk_stream_sync": (i32, [vp]),
    "nsk_device_sync": (i32, []),
    "nsk_event_create": (i32, [i32, C.POINTER(vp)]),
    "nsk_event_destroy": (i32, [vp]),
    "nsk_event_record": (i32, [vp, vp]),
    "nsk_event_wait": (i32, [vp, vp]),
    "nsk_event_sync": (i32, [vp]),
    "nsk_event_elapsed_ms": (i32, [vp, vp, C.POINTER(f32)]),
    "nsk_spin": (i32, [u64, vp]),
    "nsk_event_record_external": (i32, [vp, vp]),
    "nsk_graph_begin": (i32, [vp]),
    "nsk_graph_end": (i32, [vp, C.POINTER(vp), C.POINTER(u64)]),
    "nsk_graph_launch": (i32, [vp, vp]),
    "nsk_graph_destroy": (i32, [vp]),
    "nsk_stream_is_capturing": (i32, [vp, C.POINTER(i32)]),
    "nsk_gemm": (i32, [i32, i32, i32, i32, i32, i32, vp, i64, vp, i64, vp, i64, i32, vp, f32, vp]),
    "nsk_conv2d_fprop": (i32, [C.POINTER(ConvDesc), vp, vp, vp, i32, vp]),
    "nsk_conv2d_fprop_stats": (i32, [C.POINTER(ConvDesc), vp, vp, vp, vp, u64, C.POINTER(C.c_int), vp]),
    "nsk_wgrad_grid_cap": (i32, [i32]),
    "nsk_conv2d_dgrad": (i32, [C.POINTER(ConvDesc), vp, vp, vp, vp]),
    "nsk_conv2d_dgrad_acc": (i32, [C.POINTER(ConvDesc), vp, vp, vp, f32, vp]),
    "nsk_conv2d_dgrad_bnstats": (i32, [C.POINTER(ConvDesc), vp, vp, vp, f32, vp, vp, vp, u64, C.POINTER(i32), vp]),
    "nsk_conv2d_wgrad_workspace": (u64, [C.POINTER(ConvDesc)]),
    "nsk_conv2d_wgrad": (i32, [C.POINTER(ConvDesc), vp, vp, vp, f32, vp, u64, vp]),
    "nsk_gemm_simt": (i32, [i32, i32, i32, i32, i32, vp, i64, vp, i64, vp, i64, vp, f32, vp]),
    "nsk_fill_f32": (i32, [vp, u64, f32, vp]),
    "nsk_fill_bf16": (i32, [vp, u64, f32, vp]),
    "nsk_cast": (i32, [i32, vp, i32, vp, u64, vp]),
    "nsk_eltwise": (i32, [i32, i32, vp, vp, f32, vp, u64, vp]),
    "nsk_eltwise_bwd": (i32, [i32, i32, vp, vp, f32, vp, u64, vp]),
    "nsk_axpy": (i32, [i32, vp, vp, f32, u64, vp]),
    "nsk_bias_add": (i32, [i32, vp, vp, vp, u64, u64, vp]),
    "nsk_colsum": (i32, [i32, vp, vp, u64, u64, f32, vp]),
    "nsk_onehot": (i32, [vp, u64, i32, vp, vp, vp]),
    "nsk_check_indices": (i32, [vp, u64, i32, vp, vp]),
    "nsk_transpose_2d": (i32, [i32, vp, vp, u64, u64, vp]),
    "nsk_xent_fwd": (i32, [vp, vp, i32, i32, vp, vp, vp, vp]),
    "nsk_xent_bwd": (i32, [vp, vp, vp, i32, i32, vp, vp]),
    "nsk_sum_f32": (i32, [i32, vp, u64, vp, vp]),
    "nsk_fill_like_scalar": (i32, [vp, vp, u64, vp]),
    "nsk_argmax_correct": (i32, [vp, vp, i32, i32, vp, vp]),
    "nsk_sgd_multi": (i32, [i32, vp, vp, vp, vp, vp, f64, f64, f32, vp]),
    "nsk_adamw_multi": (i32, [i32, vp, vp, vp, vp, vp, vp, vp, f64, f64, f64, f64, f64, vp, vp]),
    "nsk_sqnorm_multi": (i32, [i32, vp, vp, vp, vp]),
    "nsk_clip_scale": (i32, [vp, f32, vp, vp]),
    "nsk_scale_multi": (i32, [i32, vp, vp, vp, vp]),
    "nsk_bn_workspace": (u64, [u64, i32]),
    "nsk_bn_fwd": (i32, [vp, vp, vp, vp, vp, u64, i32, f32, i32, vp, vp, vp, f32, vp, vp]),
    "nsk_bn_fwd_partials": (i32, [vp, i32, vp, vp, vp, vp, vp, u64, i32, f32, i32, vp, vp, vp, f32, vp, vp]),
    "nsk_bn_bwd": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, f32, u64, i32, vp, vp]),
    "nsk_bn_bwd_partials": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, f32, u64, i32, vp, vp]),
    "nsk_bn_running_update": (i32, [vp, vp, vp, u64, i32, f32, f32, vp]),
    "nsk_bn_fwd_eval": (i32, [vp, vp, vp, vp, u64, i32, f32, i32, vp, vp, vp]),
    "nsk_avgpool_fwd": (i32, [i32, vp, vp, i32, i32, i32, vp]),
    "nsk_avgpool_bwd": (i32, [vp, i32, vp, i32, i32, i32, vp]),
    "nsk_maxpool_fwd": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp]),
    "nsk_maxpool_bwd": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp]),
    "nsk_nchw_to_nhwc": (i32, [vp, vp, i32, i32, i32, i32, i32, vp]),
    "nsk_nhwc_to_nchw": (i32, [i32, vp, vp, i32, i32, i32, i32, i32, vp]),
    "nsk_im2col": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp]),
    "nsk_im2col_nchw": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp]),
    "nsk_col2im":(i32, [vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp]),
    "nsk_augment_crop_flip": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, i32, vp]),
    "nsk_embedding_fwd": (i32, [vp, vp, u64, i32, i32, i32, i32, vp, vp, vp]),
    "nsk_embedding_bwd": (i32, [vp, i32, vp, u64, i32, i32, vp, vp]),
    "nsk_gru_fwd": (i32, [vp, vp, vp, i32, i32, i32, vp, vp, vp]),
    "nsk_gru_bwd": (i32, [vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, u64, vp]),
    "nsk_gru_bwd_workspace": (u64, [i32, i32, i32]),
    "nsk_gru_tc_supported": (i32, [i32, i32]),
    "nsk_gru_trace": (i32, [vp, i32]),
    "nsk_gru_tc_workspace": (u64, [i32, i32]),
    "nsk_gru_fwd_tc": (i32, [vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, u64, vp]),
    "nsk_gru_bwd_tc": (i32, [vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, f32, vp, f32, vp, u64, vp]),
    "nsk_comm_unique_id": (i32, [vp]),
    "nsk_comm_init": (i32, [i32, i32, vp, C.POINTER(vp)]),
    "nsk_comm_destroy": (i32, [vp]),
    "nsk_allreduce": (i32, [vp, vp, u64, i32, vp]),
    "nsk_allreduce_i32": (i32, [vp, vp, u64, vp]),
    "nsk_comm_check": (i32, [vp]),
}

_lib = None
_lock = threading.Lock()


def _bundled_nccl() -> str | None:
    """Path of the libnccl.so.2 PyTorch ships (nvidia-nccl wheel), found without importing torch. One process
    holds one libnccl.so.2 and torch needs its own version, so libnskb uses the same file."""
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


def load():
    """Load libnskb.so and bind every exported symbol (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        if "NSK_NCCL_LIB" not in os.environ:  # comm.cu binds NCCL at run time: prefer PyTorch's bundled copy
            nccl = _bundled_nccl()
            if nccl:
                os.environ["NSK_NCCL_LIB"] = nccl
        lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue  # declared but not built (checked by tests/test_abi.py)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def error_for(rc: int, msg: str) -> Exception:
    if rc == 2:
        return NskTypeError(msg)
    return NskRuntimeError(msg)


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.nsk_last_error().decode(errors="replace") if _lib is not None else f"status {rc}"
        raise error_for(rc, msg)


class _Context:
    """Per-process device context: device id, compute stream, SM count."""

    def __init__(self):
        self.ready = False
        self.device = 0
        self.stream = None
        self.sm_count = 0
        self.cc = (0, 0)
        self.total_mem = 0
        self._lock = threading.Lock()

    def init(self, device: int | None = None):
        if self.ready:
            return self
        with self._lock:
            if self.ready:
                return self
            lib = load()
            dev = int(os.environ.get("LOCAL_RANK", "0")) if device is None else device
            check(lib.nsk_init(dev))
            sm, ma, mi, tot = i32(), i32(), i32(), u64()
            check(lib.nsk_device_info(C.byref(sm), C.byref(ma), C.byref(mi), C.byref(tot)))
            if ma.value != 10:
                raise NskRuntimeError(f"libnskb targets sm_100a (B200); found compute capability {ma.value}.{mi.value}")
            s = vp()
            check(lib.nsk_stream_create(C.byref(s)))
            self.device, self.stream = dev, s.value
            self.sm_count, self.cc, self.total_mem = sm.value, (ma.value, mi.value), tot.value
            self.ready = True
        return self


ctx = _Context()


def lib():
    """The bound library with the device context initialised."""
    if not ctx.ready:
        ctx.init()
    return _lib


def stream():
    if not ctx.ready:
        ctx.init()
    return ctx.stream


def sync():
    check(lib().nsk_stream_sync(stream()))
