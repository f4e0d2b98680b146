"""Training stdlib on the device: init, linear, losses, optimizers, clipping.

Drop-in counterpart of pkg/src/nsk/nn.py. Same names, signatures, defaults
(Hyperparams nn.py:22-35) and update formulas; the optimizers run as one
multi-tensor kernel over every parameter (float64 math, float32 store, as
nn.py:91-119) and also refresh the bf16 shadow weights the tensor-core
kernels read. Optimizer state lives in device buffers owned by the ParamGroup.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, autodiff
from ._lib import BF16, F32, check
from .autodiff import rec_bias_add, rec_cross_entropy, rec_matmul_t, rec_sum_loss
from .errors import NskRuntimeError
from .tensor import SCALARS, Buffer, DeviceScalar, GradCache, Pool, Tensor, tensor_from_array


@dataclass
class Hyperparams:
    learning_rate: float = 0.001
    weight_decay: float = 0.0001
    clip_norm: float = 5.0
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise NskRuntimeError(f"learning rate must be positive, got {self.learning_rate}")
        if self.clip_norm is not None and self.clip_norm <= 0:
            raise NskRuntimeError(f"clip norm must be positive, got {self.clip_norm}")


class DeviceTable:
    """A small device array of uint64 (pointer / size tables for multi-tensor kernels)."""

    def __init__(self, values):
        arr = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
        self.n = arr.size
        self.buf = Buffer(max(2 * self.n, 2), F32)
        if self.n:
            check(_lib.lib().nsk_memcpy_h2d(self.buf.ptr, arr.ctypes.data, arr.nbytes, _lib.stream()))
            _lib.sync()

    @property
    def ptr(self):
        return self.buf.ptr


class ParamGroup:
    """Named trainable tensors plus their per-parameter device optimizer state (nn.py:38-57)."""

    def __init__(self):
        self.params: list[tuple[str, Tensor]] = []
        self.state: dict[str, dict[str, Buffer]] = {}
        self.step_count = 0
        self._tables = {}
        self.grad_scale = 1.0  # data-parallel averaging (1/world) folded into the update
        self.flat = None
        self.auto_flatten = True
        self.step_dev = None
        self._scale_buf = None

    def scale_dev(self) -> Buffer:
        """Device float holding grad_scale (data-parallel 1/N), created once outside graph capture."""
        if self._scale_buf is None:
            self._scale_buf = Buffer(1, F32)
            self._scale_buf.fill(float(self.grad_scale))
        return self._scale_buf

    def add(self, name: str, tensor: Tensor) -> None:
        self.params.append((name, tensor))

    def __len__(self):
        return len(self.params)

    def _state_for(self, name: str, tensor: Tensor, keys: tuple[str, ...]) -> dict[str, Buffer]:
        st = self.state.setdefault(name, {})
        for k in keys:
            if k not in st:
                b = Buffer(tensor.numel, F32)
                b.fill(0.0)
                st[k] = b
        return st

    FLAT_ALIGN = 8  # elements: keeps every bf16 shadow view 16-byte aligned (TMA operands)

    def flatten(self, cache: GradCache, state_keys: tuple[str, ...]) -> None:
        """Relocate parameters, their gradients, optimizer state and bf16 shadows into four contiguous
        arenas sharing one layout (reverse declaration order: the order backward finalises gradients).
        The optimizer then runs as a single flat sweep and data-parallel buckets are contiguous slices."""
        for name, _t in self.params:
            if cache.buffer(name) is None:
                raise NskRuntimeError(f"missing gradient for parameter {name!r}")
        offs, total = {}, 0
        for name, t in reversed(self.params):
            offs[name] = total
            total += (t.numel + self.FLAT_ALIGN - 1) // self.FLAT_ALIGN * self.FLAT_ALIGN
        lib, st = _lib.lib(), _lib.stream()
        warena = Buffer(total, F32)
        warena.fill(0.0)
        sarena = Buffer(total, BF16)
        sarena.fill(0.0)
        for name, t in self.params:
            view = Buffer(t.numel, F32, base=warena, offset=offs[name])
            check(lib.nsk_memcpy_d2d(view.ptr, t.ptr, t.buffer.nbytes, st))
            old, t.buffer = t.buffer, view
            old.free()
            t.shadow = Buffer(t.numel, BF16, base=sarena, offset=offs[name])
            t.shadow_version = -1
        cache.flatten_with(offs, total)
        arenas = {}
        for k in state_keys:
            a = Buffer(total, F32)
            a.fill(0.0)
            for name, t in self.params:
                old = self.state.get(name, {}).get(k)
                view = Buffer(t.numel, F32, base=a, offset=offs[name])
                if old is not None:
                    check(lib.nsk_memcpy_d2d(view.ptr, old.ptr, old.nbytes, st))
                self.state.setdefault(name, {})[k] = view
            arenas[k] = a
        self.flat = {"offsets": offs, "total": total, "w": warena, "shadow": sarena, "state": arenas}
        self._tables = {}

    def _table(self, kind: str, cache: GradCache, keys: tuple[str, ...]):
        """Pointer tables (w, g, state..., shadow, numel) for the multi-tensor kernels; cached by addresses."""
        if self.flat is None and self.auto_flatten and self.params:
            self.flatten(cache, keys)
        if self.flat is not None and all(k in self.flat["state"] for k in keys) and cache.arena is not None:
            f = self.flat
            sig = (kind, "flat", f["w"].ptr, cache.arena.ptr)
            tab = self._tables.get(kind)
            if tab is None or tab[0] != sig:
                vals = {"w": [f["w"].ptr], "g": [cache.arena.ptr], "b": [f["shadow"].ptr], "n": [f["total"]]}
                for k in keys:
                    vals[k] = [f["state"][k].ptr]
                tab = (sig, {k: DeviceTable(v) for k, v in vals.items()})
                self._tables[kind] = tab
            return tab[1], 1
        return self._tensor_table(kind, cache, keys), len(self.params)

    def _tensor_table(self, kind: str, cache: GradCache, keys: tuple[str, ...]):
        cols = {"w": [], "g": [], "b": [], "n": []}
        for k in keys:
            cols[k] = []
        for name, t in self.params:
            gb = cache.buffer(name)
            if gb is None:
                raise NskRuntimeError(f"missing gradient for parameter {name!r}")
            st = self._state_for(name, t, keys)
            cols["w"].append(t.ptr)
            cols["g"].append(gb.ptr)
            for k in keys:
                cols[k].append(st[k].ptr)
            cols["b"].append(t.shadow.ptr if t.shadow is not None else 0)
            cols["n"].append(t.numel)
        sig = (kind,) + tuple(tuple(v) for v in cols.values())
        tab = self._tables.get(kind)
        if tab is None or tab[0] != sig:
            tab = (sig, {k: DeviceTable(v) for k, v in cols.items()})
            self._tables[kind] = tab
        return tab[1]

    def _after_update(self):
        for _name, t in self.params:
            t.version += 1
            if t.shadow is not None:
                t.shadow_version = t.version


def xavier_uniform_init(rows: int, cols: int, seed: int, pool: Pool, name: str | None = None) -> Tensor:
    """Uniform(-a, a), a = sqrt(6 / (rows + cols)); host RNG identical to nn.py:60-71."""
    if rows < 1 or cols < 1:
        raise NskRuntimeError(f"invalid weight shape {rows}x{cols}")
    a = math.sqrt(6.0 / (rows + cols))
    rng = np.random.default_rng(seed)
    values = rng.uniform(-a, a, size=(rows, cols)).astype(np.float32)
    if name is not None:
        return autodiff.make_param(pool, values, name)
    return tensor_from_array(pool, values)


def xavier_uniform_conv(cout: int, r: int, s: int, cin: int, seed: int, pool: Pool, name: str) -> Tensor:
    """Conv filters KRSC: a = sqrt(6 / (cin*r*s + cout*r*s)) (restated fan-in/out; see oracle/restated.py)."""
    a = math.sqrt(6.0 / (cin * r * s + cout * r * s))
    rng = np.random.default_rng(seed)
    values = rng.uniform(-a, a, size=(cout, r, s, cin)).astype(np.float32)
    return autodiff.make_param(pool, values, name)


def linear(x: Tensor, w: Tensor, b: Tensor, pool: Pool) -> Tensor:
    """y = x @ w + b broadcast over rows, fully tape-recorded (nn.py:74-76)."""
    return rec_bias_add(rec_matmul_t(x, w, pool), b, pool)


cross_entropy = rec_cross_entropy
sum_loss = rec_sum_loss


def sgd_step(group: ParamGroup, cache: GradCache, lr: float, momentum: float = 0.0) -> None:
    """v <- momentum*v + g; w <- w - lr*v (nn.py:91-99). One launch for all parameters."""
    group.step_count += 1
    tab, nt = group._table("sgd", cache, ("velocity",))
    check(_lib.lib().nsk_sgd_multi(nt, tab["w"].ptr, tab["g"].ptr, tab["velocity"].ptr,
                                   tab["b"].ptr, tab["n"].ptr, float(lr), float(momentum),
                                   float(group.grad_scale), _lib.stream()))
    group._after_update()


def adamw_step(group: ParamGroup, cache: GradCache, hp: Hyperparams, grad_scale_dev: int | None = None,
               apply_group_scale: bool = True) -> None:
    """Decoupled weight decay, then the bias-corrected Adam update (nn.py:102-119)."""
    group.step_count += 1
    tab, nt = group._table("adamw", cache, ("m", "v"))
    if group.step_dev is None:  # device copy of step_count: captured graphs replay with t = 1, 2, ...
        group.step_dev = Buffer(1, F32)
        arr = np.array([group.step_count - 1], np.int32)
        check(_lib.lib().nsk_memcpy_h2d(group.step_dev.ptr, arr.ctypes.data, 4, _lib.stream()))
        _lib.sync()
    scale_ptr = grad_scale_dev
    if scale_ptr is None and apply_group_scale and group.grad_scale != 1.0:
        scale_ptr = group.scale_dev().ptr
    check(_lib.lib().nsk_adamw_multi(nt, tab["w"].ptr, tab["g"].ptr, tab["m"].ptr, tab["v"].ptr,
                                     tab["b"].ptr, tab["n"].ptr, group.step_dev.ptr, float(hp.learning_rate),
                                     float(hp.weight_decay), float(hp.beta1), float(hp.beta2), float(hp.epsilon),
                                     scale_ptr, _lib.stream()))
    group._after_update()


class _ClipState:
    def __init__(self):
        self.sq = None
        self.tables = {}


_CLIP = _ClipState()


def clip_grad_norm(cache: GradCache, max_norm: float) -> DeviceScalar:
    """Scale all cached gradients so their global L2 norm is at most max_norm (nn.py:122-139).

    Returns the applied scale as a DeviceScalar (``float()`` reads it); the
    norm is accumulated in float64 and gradients are scaled in float32.
    """
    if max_norm <= 0:
        raise NskRuntimeError(f"clip norm must be positive, got {max_norm}")
    if cache.arena is not None and len(cache.offsets) == len(cache.grads):
        ptrs, sizes = [cache.arena.ptr], [cache.arena.capacity]  # padding slots are zero
    else:
        names = list(cache.grads.keys())
        ptrs = [cache.grads[n].ptr for n in names]
        sizes = [cache.grads[n].capacity for n in names]
    key = (tuple(ptrs), tuple(sizes))
    tab = _CLIP.tables.get(key)
    if tab is None:
        tab = (DeviceTable(ptrs), DeviceTable(sizes))
        _CLIP.tables[key] = tab
    if _CLIP.sq is None:
        _CLIP.sq = Buffer(2 * 1025, F32)
    slot = SCALARS.take()
    lib = _lib.lib()
    st = _lib.stream()
    check(lib.nsk_sqnorm_multi(len(ptrs), tab[0].ptr, tab[1].ptr, _CLIP.sq.ptr, st))
    check(lib.nsk_clip_scale(_CLIP.sq.ptr, float(max_norm), SCALARS.ptr(slot), st))
    check(lib.nsk_scale_multi(len(ptrs), tab[0].ptr, tab[1].ptr, SCALARS.ptr(slot), st))
    return DeviceScalar(slot)


def xavier_values(rows: int, cols: int, seed: int) -> np.ndarray:
    """The float32 values xavier_uniform_init draws (nn.py:60-71), without making a tensor."""
    a = math.sqrt(6.0 / (rows + cols))
    return np.random.default_rng(seed).uniform(-a, a, size=(rows, cols)).astype(np.float32)


def scale_grads(cache: GradCache, scale_dev: Buffer) -> None:
    """In-place g *= scale for every cached gradient (data-parallel averaging ahead of clipping)."""
    if cache.arena is not None and len(cache.offsets) == len(cache.grads):
        ptrs, sizes = [cache.arena.ptr], [cache.arena.capacity]
    else:
        ptrs = [b.ptr for b in cache.grads.values()]
        sizes = [b.capacity for b in cache.grads.values()]
    key = ("scale",) + tuple(ptrs)
    tab = _CLIP.tables.get(key)
    if tab is None:
        tab = (DeviceTable(ptrs), DeviceTable(sizes))
        _CLIP.tables[key] = tab
    check(_lib.lib().nsk_scale_multi(len(ptrs), tab[0].ptr, tab[1].ptr, scale_dev.ptr, _lib.stream()))
