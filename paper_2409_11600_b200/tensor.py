"""Device tensor engine: pooled device buffers, tensor handles, CUDA kernels.

Drop-in counterpart of pkg/src/nsk/tensor.py. The Pool keeps the reference's
contract exactly -- exact-size keys, LIFO reuse, unbounded growth, no zeroing,
``enabled=False`` baseline, ``poison=True`` NaN fill on release, the same
``fresh/hits/released`` counters (tensor.py:54-113) -- but its buffers are
HBM blocks from libnskb's size-class caching arena instead of mmap pages.
Keys are (numel, dtype) because activations are bf16 NHWC while parameters and
gradients stay float32. Every kernel fully overwrites its output buffer
(tensor.py:6-8), so poisoned pooled memory never leaks into results.

Host reads (``Tensor.data``, ``item``) synchronise the compute stream; nothing
inside a training step does, so a warm step can be captured as a CUDA graph.
"""

from __future__ import annotations

import ctypes as C
import os
import numbers
import threading

import numpy as np

from . import _lib
from ._lib import BF16, DTYPE_SIZE, F32, check
from .errors import NskRuntimeError, NskTypeError

ELEMENTWISE_KINDS = frozenset(
    {"add", "sub", "hadamard", "scalar-add", "scalar-mul", "relu", "sigmoid", "tanh", "neg"}
)
EW_CODE = {"add": 0, "sub": 1, "hadamard": 2, "scalar-add": 3, "scalar-mul": 4, "relu": 5, "sigmoid": 6,
           "tanh": 7, "neg": 8, "copy": 9}

MATMUL_PRECISION = os.environ.get("NSK_MATMUL_PRECISION", "tf32")  # "tf32" (tcgen05) | "fp32" (fp64-accum SIMT)
_TC_MIN_WORK = 1 << 24  # below this M*N*K the exact SIMT kernel costs only microseconds


class _GrowBuffer:
    """Grow-only float32 scratch (stream-ordered reuse by consecutive kernels)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int):
        if self.buf is None or self.buf.nbytes < nbytes:
            self.buf = Buffer((max(nbytes, 1 << 20) + 3) // 4, F32)
        return self.buf


_TRANSPOSE_WS = _GrowBuffer()


def _np_dtype(dtype):
    return np.float32 if dtype == F32 else np.uint16


# --- memory -------------------------------------------------------------------------

class Buffer:
    """A flat device allocation of ``capacity`` elements of ``dtype``.

    Views (``base`` set) alias a slice of a parent allocation (the flat
    gradient / parameter arenas) and never free.
    """

    __slots__ = ("capacity", "dtype", "ptr", "origin", "in_pool", "base", "__weakref__")

    def __init__(self, capacity: int, dtype: int = F32, base: "Buffer | None" = None, offset: int = 0):
        self.capacity = int(capacity)
        self.dtype = dtype
        self.origin = "fresh"
        self.in_pool = False
        self.base = base
        if base is not None:
            self.ptr = base.ptr + offset * DTYPE_SIZE[dtype]
            return
        lib = _lib.lib()
        p = C.c_void_p()
        rc = lib.nsk_arena_alloc(max(self.capacity, 1) * DTYPE_SIZE[dtype], _lib.stream(), C.byref(p))
        if rc == 1:
            lib.nsk_last_error()
            raise NskRuntimeError(f"out of memory: requested {capacity} elements") from None
        check(rc)
        self.ptr = p.value

    @property
    def nbytes(self) -> int:
        return self.capacity * DTYPE_SIZE[self.dtype]

    def host(self) -> np.ndarray:
        """Synchronous copy to a host array (bf16 is returned as float32)."""
        out = np.empty(self.capacity, dtype=_np_dtype(self.dtype))
        if self.capacity:
            check(_lib.lib().nsk_memcpy_d2h(out.ctypes.data, self.ptr, self.nbytes, _lib.stream()))
            _lib.sync()
        if self.dtype == BF16:
            return (out.astype(np.uint32) << 16).view(np.float32)
        return out

    @property
    def storage(self) -> np.ndarray:
        """The contents as a host array (reference tensor.py:40-48 exposes the memory itself): item assignment
        on the returned array (``storage[:] = v``, ``storage[i] = v``) is written back to the device."""
        view = self.host().view(_StorageView)
        view._dev = self
        return view

    def upload(self, array) -> None:
        arr = np.ascontiguousarray(np.asarray(array, dtype=np.float32).reshape(-1))
        if arr.size != self.capacity:
            raise NskRuntimeError(f"upload of {arr.size} elements into a buffer of {self.capacity}")
        if self.dtype == BF16:
            arr = to_bf16_bits(arr)
        check(_lib.lib().nsk_memcpy_h2d(self.ptr, arr.ctypes.data, self.nbytes, _lib.stream()))
        _lib.sync()

    def fill(self, value: float) -> None:
        lib = _lib.lib()
        if self.dtype == F32:
            check(lib.nsk_fill_f32(self.ptr, self.capacity, value, _lib.stream()))
        else:
            check(lib.nsk_fill_bf16(self.ptr, self.capacity, value, _lib.stream()))

    def free(self) -> None:
        if self.base is None and self.ptr:
            check(_lib.lib().nsk_arena_free(self.ptr, _lib.stream()))
        self.ptr = 0

    def __del__(self):
        try:
            if self.base is None and self.ptr and _lib._lib is not None:
                _lib._lib.nsk_arena_free(self.ptr, _lib.ctx.stream)
        except Exception:  # interpreter shutdown
            pass

    def __repr__(self):
        return f"Buffer(capacity={self.capacity}, dtype={_lib.DTYPE_NAME[self.dtype]}, origin={self.origin})"


class _StorageView(np.ndarray):
    """Host copy of a device Buffer whose item assignment writes the whole copy back (Buffer.storage)."""

    _dev = None

    def __array_finalize__(self, obj):
        self._dev = None  # slices and results of arithmetic are plain host values

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        if self._dev is not None:
            self._dev.upload(self.view(np.ndarray))


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round-to-nearest-even (matches __float2bfloat16_rn)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(a.reshape(-1)) if a.ndim else np.isnan(a)
    if np.any(nan):
        r = r.reshape(-1)
        r[nan.reshape(-1)] = 0x7FC0
        r = r.reshape(u.shape)
    return r


def round_bf16(a) -> np.ndarray:
    """Round float values to the nearest bf16 (returned as float32)."""
    bits = to_bf16_bits(np.asarray(a, dtype=np.float32))
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _pool_key(numel: int, dtype: int):
    return numel if dtype == F32 else (numel, dtype)


class Pool:
    """Size-keyed free lists of reusable device buffers (reference tensor.py:54-113)."""

    def __init__(self, enabled: bool = True, poison: bool = False):
        self.enabled = enabled
        self.poison = poison
        # keyed by element count exactly as the reference (tensor.py:78) for float32; (numel, dtype) otherwise
        self.free_lists: dict[int | tuple[int, int], list[Buffer]] = {}
        self.fresh_allocations = 0
        self.pool_hits = 0
        self.releases = 0
        self._lock = threading.Lock()

    def acquire(self, numel: int, dtype: int = F32) -> Buffer:
        if numel < 1:
            raise NskRuntimeError(f"cannot allocate a buffer of {numel} elements")
        key = _pool_key(numel, dtype)
        if self.enabled:
            with self._lock:
                free = self.free_lists.get(key)
                if free:
                    buf = free.pop()
                    buf.in_pool = False
                    buf.origin = "pooled"
                    self.pool_hits += 1
                    return buf
                self.fresh_allocations += 1
        else:
            with self._lock:
                self.fresh_allocations += 1
        return Buffer(numel, dtype)

    def release(self, buffer: Buffer) -> None:
        from .side import SIDE

        if SIDE.defer(self, buffer):  # read by an in-flight side-stream kernel: released at the join
            return
        with self._lock:
            if buffer.in_pool:
                raise NskRuntimeError("double release of a pooled buffer")
            self.releases += 1
            if not self.enabled:
                buffer.free()
                return
            if self.poison:
                buffer.fill(float("nan"))
            buffer.in_pool = True
            self.free_lists.setdefault(_pool_key(buffer.capacity, buffer.dtype), []).append(buffer)

    def free_total(self) -> int:
        with self._lock:
            return sum(len(v) for v in self.free_lists.values())

    def stats(self) -> dict[str, int]:
        with self._lock:
            return {"fresh": self.fresh_allocations, "hits": self.pool_hits, "released": self.releases}


class ScalarSlots:
    """Device ring of float32 slots holding snapshots of released 1-element tensors.

    The reference snapshots ``storage[0]`` into a Python float on release
    (tensor.py:200-208), a host sync. Here the value is copied device-to-device
    into a slot and read lazily by ``item()``, so the copy can live inside a
    captured step graph.
    """

    SIZE = 1 << 16

    def __init__(self):
        self.buf = None
        self.next = 0
        self._lock = threading.Lock()

    def take(self) -> int:
        with self._lock:
            if self.buf is None:
                self.buf = Buffer(self.SIZE, F32)
            i = self.next
            self.next = (self.next + 1) % self.SIZE
            return i

    def ptr(self, i: int) -> int:
        return self.buf.ptr + 4 * i

    def read(self, i: int) -> float:
        out = np.empty(1, np.float32)
        check(_lib.lib().nsk_memcpy_d2h(out.ctypes.data, self.ptr(i), 4, _lib.stream()))
        _lib.sync()
        return float(out[0])


SCALARS = ScalarSlots()


class DeviceScalar:
    """A float that lives on the device until asked for (loss values, clip scales)."""

    __slots__ = ("slot",)

    def __init__(self, slot: int):
        self.slot = slot

    @property
    def ptr(self) -> int:
        return SCALARS.ptr(self.slot)

    def __float__(self):
        return SCALARS.read(self.slot)

    def __repr__(self):
        return f"DeviceScalar({float(self):g})"

    # arithmetic / comparison read the value (a sync), so callers written against the reference's plain floats
    # (nn.clip_grad_norm returns the scale, nn.py:122-139) keep working
    def __eq__(self, other):
        return float(self) == other

    def __ne__(self, other):
        return float(self) != other

    def __lt__(self, other):
        return float(self) < other

    def __le__(self, other):
        return float(self) <= other

    def __gt__(self, other):
        return float(self) > other

    def __ge__(self, other):
        return float(self) >= other

    __hash__ = object.__hash__

    def __add__(self, other):
        return float(self) + other

    __radd__ = __add__

    def __sub__(self, other):
        return float(self) - other

    def __rsub__(self, other):
        return other - float(self)

    def __mul__(self, other):
        return float(self) * other

    __rmul__ = __mul__

    def __truediv__(self, other):
        return float(self) / other

    def __rtruediv__(self, other):
        return other / float(self)

    def __neg__(self):
        return -float(self)

    def __abs__(self):
        return abs(float(self))

    def __bool__(self):
        return bool(float(self))


numbers.Real.register(DeviceScalar)


# --- tensors --------------------------------------------------------------------------

class Tensor:
    """A shape-tagged view over a pooled device buffer (reference tensor.py:116-170).

    Extra slots: ``dtype`` (F32 or BF16), ``host_src`` (the host array a data
    tensor was made from, so host-side index checks need no sync), ``shadow``
    (bf16 copy of a float32 parameter read by tensor-core kernels),
    ``version`` (bumped whenever a parameter's values change), ``bn_partials``
    (channel statistics a conv emitted for the BatchNorm that consumes it) and ``bnb_partials`` (on a
    gradient: the BatchNorm-backward statistics the dgrad that completed it emitted, see layers._r_conv2d).
    """

    __slots__ = ("shape", "buffer", "param_name", "node", "grad", "refs", "_scalar", "dtype", "host_src",
                 "shadow", "shadow_version", "version", "bn_partials", "bnb_partials", "__weakref__")

    def __init__(self, shape: tuple[int, ...], buffer: Buffer, param_name: str | None = None):
        numel = 1
        for d in shape:
            if d < 1:
                raise NskRuntimeError(f"invalid tensor dimension {d}")
            numel *= d
        if numel != buffer.capacity:
            raise NskRuntimeError(f"shape {shape} needs {numel} elements, buffer holds {buffer.capacity}")
        self.shape = tuple(int(d) for d in shape)
        self.buffer: Buffer | None = buffer
        self.param_name = param_name
        self.node = None
        self.grad: Tensor | None = None
        self.refs = 0
        self._scalar = None
        self.dtype = buffer.dtype
        self.host_src = None
        self.shadow = None
        self.shadow_version = -1
        self.version = 0
        self.bn_partials = None
        self.bnb_partials = None  # (gradient tensors) BatchNorm-backward partials a dgrad emitted with it

    @property
    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def rank(self) -> int:
        return len(self.shape)

    @property
    def ptr(self) -> int:
        if self.buffer is None:
            raise NskRuntimeError("tensor buffer was reclaimed by backward()")
        return self.buffer.ptr

    @property
    def data(self) -> np.ndarray:
        """Host copy of the values (synchronises the compute stream)."""
        if self.buffer is None:
            raise NskRuntimeError("tensor buffer was reclaimed by backward()")
        return self.buffer.host().reshape(self.shape)

    def item(self) -> float:
        if self.buffer is None:
            if self._scalar is not None:
                return float(self._scalar)
            raise NskRuntimeError("tensor buffer was reclaimed by backward()")
        if self.numel != 1:
            raise NskRuntimeError(f"item() needs a 1-element tensor, got shape {self.shape}")
        return float(self.buffer.host()[0])

    def bf16_ptr(self, pool: "Pool | None" = None) -> int:
        """Device pointer of a bf16 copy (self if already bf16; refreshed shadow for f32 params)."""
        if self.dtype == BF16:
            return self.ptr
        if self.shadow is None:
            self.shadow = Buffer(self.numel, BF16)
        if self.shadow_version != self.version:
            check(_lib.lib().nsk_cast(F32, self.ptr, BF16, self.shadow.ptr, self.numel, _lib.stream()))
            self.shadow_version = self.version
        return self.shadow.ptr

    def __repr__(self):
        name = f", param={self.param_name}" if self.param_name else ""
        if self.buffer is None:
            body = "<reclaimed>" if self._scalar is None else f"<reclaimed value={float(self._scalar):g}>"
        else:
            body = np.array2string(self.data, precision=4, suppress_small=True)
        return f"Tensor(shape={list(self.shape)}{name}, dtype={_lib.DTYPE_NAME[self.dtype]}) {body}"


MAX_RANK = 4


def tensor_from_array(pool: Pool, array, param_name: str | None = None, dtype: int = F32) -> Tensor:
    """Copy host data into a pool-acquired device buffer (reference tensor.py:181-190; rank <= 4 here)."""
    arr = np.asarray(array, dtype=np.float32)
    if arr.ndim == 0:
        arr = arr.reshape(1)
    if arr.ndim > MAX_RANK:
        raise NskRuntimeError(f"rank {arr.ndim} tensors are not supported")
    buf = pool.acquire(arr.size, dtype)
    try:
        buf.upload(arr)
    except Exception:
        pool.release(buf)
        raise
    return Tensor(tuple(arr.shape), buf, param_name=param_name)


def empty_tensor(pool: Pool, shape: tuple[int, ...], dtype: int = F32) -> Tensor:
    numel = 1
    for d in shape:
        numel *= d
    return Tensor(shape, pool.acquire(numel, dtype))


def release_tensor(pool: Pool, t: Tensor) -> None:
    """Return a tensor's buffer to the pool, snapshotting 1-element values on the device."""
    if t.buffer is None:
        return
    if t.numel == 1 and t.dtype == F32:
        slot = SCALARS.take()
        check(_lib.lib().nsk_memcpy_d2d(SCALARS.ptr(slot), t.buffer.ptr, 4, _lib.stream()))
        t._scalar = DeviceScalar(slot)
    buf = t.buffer
    t.buffer = None
    pool.release(buf)


def fill_tensor(t: Tensor, value: float) -> Tensor:
    t.buffer.fill(value)
    return t


# --- kernels -----------------------------------------------------------------------------
class _Operands:
    """Device pointers of GEMM operands in ``dtype``: tensors already in it as-is, float32 parameters
    via their bf16 shadow, anything else through pooled cast copies released on exit."""

    def __init__(self, pool: Pool, dtype: int, *tensors: Tensor):
        self.pool = pool
        self.dtype = dtype
        self.tensors = tensors
        self.temps = []

    def __enter__(self):
        ptrs = []
        for t in self.tensors:
            if t.dtype == self.dtype:
                ptrs.append(t.ptr)
            elif self.dtype == BF16 and t.param_name is not None:
                ptrs.append(t.bf16_ptr())
            else:
                tmp = empty_tensor(self.pool, t.shape, self.dtype)
                check(_lib.lib().nsk_cast(t.dtype, t.ptr, self.dtype, tmp.ptr, t.numel, _lib.stream()))
                self.temps.append(tmp)
                ptrs.append(tmp.ptr)
        return ptrs

    def __exit__(self, *exc):
        for t in self.temps:
            release_tensor(self.pool, t)
        return False


def _gemm(a_ptr, a_mn, lda, b_ptr, b_mn, ldb, M, N, K, out_ptr, ldc, dtype=F32, bias_ptr=None, beta=0.0,
          out_f32=True):
    """C[M,N] = A(M,K) . B(N,K)^T, dispatching tcgen05 (tf32/bf16) or the exact SIMT kernel."""
    lib = _lib.lib()
    st = _lib.stream()
    esz = DTYPE_SIZE[dtype]
    aligned = (lda * esz) % 16 == 0 and (ldb * esz) % 16 == 0 and a_ptr % 16 == 0 and b_ptr % 16 == 0
    if dtype == BF16:
        if not aligned:
            raise NskRuntimeError("bf16 GEMM operands must have 16-byte aligned rows")
        check(lib.nsk_gemm(BF16, a_mn, b_mn, M, N, K, a_ptr, lda, b_ptr, ldb, out_ptr, ldc, int(out_f32),
                           bias_ptr, beta, st))
        return
    use_tc = MATMUL_PRECISION == "tf32" and aligned and M * N * K >= _TC_MIN_WORK
    if use_tc and (a_mn or b_mn):
        # MN-major float32 operands (weight / input gradients of a large classifier): transpose them to
        # K-major once (a memory pass) and stay on the tf32 tensor cores instead of the SIMT kernel
        ws = _TRANSPOSE_WS.get(4 * ((M * K if a_mn else 0) + (N * K if b_mn else 0)))
        p = ws.ptr
        if a_mn:  # A stored [K, M] with row pitch lda -> [M, K]
            if lda != M:
                use_tc = False
            else:
                check(lib.nsk_transpose_2d(F32, a_ptr, p, K, M, st))
                a_ptr, lda, a_mn, p = p, K, 0, p + 4 * M * K
        if b_mn and use_tc:
            if ldb != N:
                use_tc = False
            else:
                check(lib.nsk_transpose_2d(F32, b_ptr, p, K, N, st))
                b_ptr, ldb, b_mn = p, K, 0
        if use_tc and ((lda * 4) % 16 or (ldb * 4) % 16):
            use_tc = False
    if use_tc and not a_mn and not b_mn:
        check(lib.nsk_gemm(F32, 0, 0, M, N, K, a_ptr, lda, b_ptr, ldb, out_ptr, ldc, 1, bias_ptr, beta, st))
    else:
        check(lib.nsk_gemm_simt(a_mn, b_mn, M, N, K, a_ptr, lda, b_ptr, ldb, out_ptr, ldc, bias_ptr, beta, st))


def _matmul(pool: Pool, a: Tensor, a_mn: int, lda: int, b: Tensor, b_mn: int, ldb: int, M: int, N: int, K: int,
            out: Tensor, ldc: int, beta: float = 0.0) -> None:
    """Run in bf16 on the tensor cores when an operand is bf16 and rows are 16-byte aligned, else in float32."""
    dtype = BF16 if (BF16 in (a.dtype, b.dtype) and (lda * 2) % 16 == 0 and (ldb * 2) % 16 == 0) else F32
    with _Operands(pool, dtype, a, b) as (ap, bp):
        _gemm(ap, a_mn, lda, bp, b_mn, ldb, M, N, K, out.ptr, ldc, dtype=dtype, beta=beta)


def matmul_t(x: Tensor, w: Tensor, pool: Pool) -> Tensor:
    """y[i, j] = sum_c x[i, c] * w[j, c] (reference tensor.py:213-229)."""
    if x.rank != 2 or w.rank != 2:
        raise NskTypeError(f"@ needs two matrices, got shapes {list(x.shape)} and {list(w.shape)}")
    m, k = x.shape
    n, k2 = w.shape
    if k != k2:
        raise NskTypeError(
            f"@ shape mismatch: {m}x{k} @ {n}x{k2} (columns must agree; the right operand is transposed)")
    out = empty_tensor(pool, (m, n))
    _matmul(pool, x, 0, k, w, 0, k, m, n, k, out, n)
    return out


def matmul_nn(g: Tensor, w: Tensor, pool: Pool) -> Tensor:
    """dx = g . w  (g [m,n], w [n,k] -> [m,k]); the plain_matmul of gradient_rule (tensor.py:232-234)."""
    m, n = g.shape
    n2, k = w.shape
    out = empty_tensor(pool, (m, k))
    _matmul(pool, g, 0, n, w, 1, k, m, k, n, out, k)
    return out


def matmul_tn(g: Tensor, x: Tensor, pool: Pool, out: Tensor | None = None, beta: float = 0.0) -> Tensor:
    """dw = g^T . x  (g [m,n], x [m,k] -> [n,k]) with optional accumulation into ``out``."""
    m, n = g.shape
    m2, k = x.shape
    if out is None:
        out = empty_tensor(pool, (n, k))
    _matmul(pool, g, 1, n, x, 1, k, n, k, m, out, k, beta=beta)
    return out


def elementwise(kind: str, a: Tensor, b, pool: Pool) -> Tensor:
    """Elementwise op into a pooled output buffer (reference tensor.py:247-283)."""
    if kind not in ELEMENTWISE_KINDS:
        raise NskRuntimeError(f"unknown elementwise op {kind!r}")
    bptr = None
    scalar = 0.0
    if kind in ("add", "sub", "hadamard"):
        if not isinstance(b, Tensor):
            raise NskTypeError(f"{kind} needs two tensors")
        if a.shape != b.shape:
            raise NskTypeError(f"{kind} shape mismatch: {list(a.shape)} vs {list(b.shape)}")
        if a.dtype != b.dtype:
            raise NskTypeError(f"{kind} dtype mismatch")
        bptr = b.ptr
    elif kind in ("scalar-add", "scalar-mul"):
        scalar = float(np.float32(b))
    out = empty_tensor(pool, a.shape, a.dtype)
    check(_lib.lib().nsk_eltwise(EW_CODE[kind], a.dtype, a.ptr, bptr, scalar, out.ptr, a.numel, _lib.stream()))
    return out


def eltwise_bwd(kind: str, g: Tensor, saved: Tensor | None, pool: Pool, scalar: float = 0.0) -> Tensor:
    out = empty_tensor(pool, g.shape, g.dtype)
    check(_lib.lib().nsk_eltwise_bwd(EW_CODE[kind], g.dtype, g.ptr, None if saved is None else saved.ptr,
                                     scalar, out.ptr, g.numel, _lib.stream()))
    return out


def bias_add(x: Tensor, b: Tensor, pool: Pool) -> Tensor:
    """Add a rank-1 bias across every row (reference tensor.py:286-296); NHWC tensors add per channel."""
    if x.rank < 2 or b.rank != 1:
        raise NskTypeError(
            f"bias add needs a matrix and a vector, got shapes {list(x.shape)} and {list(b.shape)}")
    if x.shape[-1] != b.shape[0]:
        raise NskTypeError(f"bias length {b.shape[0]} does not match {x.shape[-1]} columns")
    out = empty_tensor(pool, x.shape, x.dtype)
    cols = x.shape[-1]
    check(_lib.lib().nsk_bias_add(x.dtype, x.ptr, b.ptr, out.ptr, x.numel // cols, cols, _lib.stream()))
    return out


def colsum(g: Tensor, pool: Pool, out: Tensor | None = None, beta: float = 0.0) -> Tensor:
    cols = g.shape[-1]
    if out is None:
        out = empty_tensor(pool, (cols,))
    check(_lib.lib().nsk_colsum(g.dtype, g.ptr, out.ptr, g.numel // cols, cols, beta, _lib.stream()))
    return out


def check_index_values(values: np.ndarray, classes: int, what: str) -> None:
    """Host-side range check with the reference's messages (tensor.py:308-313, autodiff.py:235-239)."""
    v = np.asarray(values, dtype=np.float32).reshape(-1)
    bad = ~((v >= 0) & (v < classes) & (v == np.floor(v)))
    if bad.any():
        row = int(np.argmax(bad))
        if what == "onehot":
            raise NskRuntimeError(f"onehot index {float(v[row]):g} out of range [0, {classes}) at row {row}")
        raise NskRuntimeError(f"target {float(v[row]):g} out of range [0, {classes}) at row {row}")


def device_index_check(idx: Tensor, classes: int, what: str) -> None:
    """Range check of device-resident indices: uses the host source when known, else a flagged kernel + sync."""
    if idx.host_src is not None:
        check_index_values(idx.host_src, classes, what)
        return
    flag = ERRFLAG.reset()
    check(_lib.lib().nsk_check_indices(idx.ptr, idx.numel, classes, flag, _lib.stream()))
    row = ERRFLAG.read()
    if row is not None:
        check_index_values(idx.data.reshape(-1), classes, what)


class _ErrFlag:
    """A device int used by kernels to report the first bad row (INT_MAX = none)."""

    def __init__(self):
        self.buf = None

    def reset(self) -> int:
        if self.buf is None:
            self.buf = Buffer(1, F32)
            self._init = np.array([2**31 - 1], dtype=np.int32)
        check(_lib.lib().nsk_memcpy_h2d(self.buf.ptr, self._init.ctypes.data, 4, _lib.stream()))
        return self.buf.ptr

    def read(self):
        out = np.empty(1, np.int32)
        check(_lib.lib().nsk_memcpy_d2h(out.ctypes.data, self.buf.ptr, 4, _lib.stream()))
        _lib.sync()
        v = int(out[0])
        return None if v == 2**31 - 1 else v


ERRFLAG = _ErrFlag()


def onehot(indices: Tensor, classes: int, pool: Pool) -> Tensor:
    """Encode integer-valued entries of a rank-1 tensor as one-hot rows (reference tensor.py:299-317)."""
    if indices.rank != 1:
        raise NskTypeError(f"onehot needs a rank-1 tensor, got shape {list(indices.shape)}")
    classes = int(classes)
    if classes < 1:
        raise NskRuntimeError(f"onehot needs at least 1 class, got {classes}")
    device_index_check(indices, classes, "onehot")
    m = indices.shape[0]
    out = empty_tensor(pool, (m, classes))
    check(_lib.lib().nsk_onehot(indices.ptr, m, classes, out.ptr, None, _lib.stream()))
    return out


# --- gradient cache ---------------------------------------------------------------------------

class GradCache:
    """Persistent per-parameter float32 gradient buffers (reference tensor.py:322-367).

    ``flatten`` moves every cached gradient into one contiguous arena (in a
    caller-chosen order) so the optimizer and the data-parallel bucketed
    all-reduce see a single flat buffer; per-parameter buffers become views.
    """

    def __init__(self):
        self.grads: dict[str, Buffer] = {}
        self.shapes: dict[str, tuple[int, ...]] = {}
        self.dirty: set[str] = set()
        self.arena: Buffer | None = None
        self.offsets: dict[str, int] = {}
        self.hooks = []  # called as hook(name) after a parameter's gradient became final for this backward
        self._lock = threading.Lock()

    def _ensure(self, name: str, shape) -> Buffer:
        buf = self.grads.get(name)
        if buf is None:
            numel = 1
            for d in shape:
                numel *= d
            buf = Buffer(numel, F32)
            buf.fill(0.0)
            self.grads[name] = buf
            self.shapes[name] = tuple(shape)
        elif self.shapes[name] != tuple(shape):
            raise NskRuntimeError(
                f"gradient shape {list(shape)} does not match cached {list(self.shapes[name])} for parameter {name!r}")
        return buf

    def accumulate(self, param_name: str, grad: Tensor) -> None:
        with self._lock:
            buf = self._ensure(param_name, grad.shape)
            if grad.dtype == F32:
                check(_lib.lib().nsk_axpy(F32, buf.ptr, grad.ptr, 1.0, grad.numel, _lib.stream()))
            else:
                tmp = Buffer(grad.numel, F32)
                check(_lib.lib().nsk_cast(BF16, grad.ptr, F32, tmp.ptr, grad.numel, _lib.stream()))
                check(_lib.lib().nsk_axpy(F32, buf.ptr, tmp.ptr, 1.0, grad.numel, _lib.stream()))
            self.dirty.add(param_name)

    def sink(self, param_name: str, shape) -> Buffer:
        """The buffer a gradient kernel may accumulate into directly (beta = 1)."""
        with self._lock:
            buf = self._ensure(param_name, shape)
            self.dirty.add(param_name)
            return buf

    def get(self, param_name: str) -> np.ndarray | None:
        with self._lock:
            buf = self.grads.get(param_name)
            if buf is None:
                return None
            return buf.host().reshape(self.shapes[param_name])

    def buffer(self, param_name: str) -> Buffer | None:
        return self.grads.get(param_name)

    def zero_after_step(self) -> None:
        with self._lock:
            if self.arena is not None and len(self.offsets) == len(self.grads):
                self.arena.fill(0.0)
            else:
                for buf in self.grads.values():
                    buf.fill(0.0)
            self.dirty.clear()

    def flatten(self, order: list[str]) -> Buffer:
        """Re-home gradients into one arena laid out in ``order`` (16-byte aligned slots)."""
        offs, total = {}, 0
        for name in order:
            if name not in self.grads:
                continue
            offs[name] = total
            total += (self.grads[name].capacity + 3) // 4 * 4
        return self.flatten_with(offs, total)

    def flatten_with(self, offs: dict[str, int], total: int) -> Buffer:
        """Re-home gradients into one arena of ``total`` floats at the given element offsets."""
        with self._lock:
            arena = Buffer(max(total, 1), F32)
            arena.fill(0.0)
            lib = _lib.lib()
            for name, off in offs.items():
                old = self.grads[name]
                view = Buffer(old.capacity, F32, base=arena, offset=off)
                check(lib.nsk_memcpy_d2d(view.ptr, old.ptr, old.nbytes, _lib.stream()))
                self.grads[name] = view
            self.arena, self.offsets = arena, offs
            return arena

    def __len__(self):
        return len(self.grads)
