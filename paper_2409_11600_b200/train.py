"""The public training-step API: host batch in, loss out, one CUDA graph per step.

A step is exactly the reference training loop body (pkg/README.md example;
builtins.py:146-169): forward through the tape, ``cross_entropy``,
``backward()``, the optimizer step, ``zero_grad()``. The first ``warmup``
steps run eagerly; they warm the Pool so every later step acquires the same
buffers in the same order (the reference's warm-pool invariant, SPEC.md:344,
test_autodiff.py:247-269). The next step is captured once as a CUDA graph and
replayed thereafter -- the per-op host bookkeeping (~8 + 15 us per op in the
reference) disappears from the steady state.

Inputs travel host -> pinned staging -> device on the compute stream before
the graph launch; the loss is read back from a device scalar slot.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, autodiff, nn
from ._lib import BF16, F32, check
from .autodiff import backward, data_from_device
from .errors import NskRuntimeError
from .tensor import SCALARS, Buffer, DeviceScalar, Tensor, check_index_values


class PinnedArray:
    """A page-locked host array (cudaHostAlloc) for async H2D staging."""

    def __init__(self, shape, dtype=np.float32):
        self.shape = tuple(shape)
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(_lib.lib().nsk_pinned_alloc(max(nbytes, 1), C.byref(p)))
        self.ptr = p.value
        self.nbytes = nbytes
        raw = (C.c_char * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(raw, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def __del__(self):
        try:
            if self.ptr and _lib._lib is not None:
                _lib._lib.nsk_pinned_free(self.ptr)
        except Exception:
            pass


class StepGraph:
    """A captured step: replay with ``launch``."""

    def __init__(self, exec_handle: int, nodes: int):
        self.exec = exec_handle
        self.nodes = nodes

    def launch(self):
        check(_lib.lib().nsk_graph_launch(self.exec, _lib.stream()))

    def __del__(self):
        try:
            if self.exec and _lib._lib is not None:
                _lib._lib.nsk_graph_destroy(self.exec)
        except Exception:
            pass


def capture(fn):
    """Run ``fn`` under stream capture and return (StepGraph, fn's result). Nothing executes yet."""
    lib = _lib.lib()
    st = _lib.stream()
    check(lib.nsk_graph_begin(st))
    try:
        result = fn()
    except BaseException:
        ex, n = C.c_void_p(), C.c_uint64()
        lib.nsk_graph_end(st, C.byref(ex), C.byref(n))
        if ex.value:
            lib.nsk_graph_destroy(ex.value)
        raise
    ex, n = C.c_void_p(), C.c_uint64()
    check(lib.nsk_graph_end(st, C.byref(ex), C.byref(n)))
    return StepGraph(ex.value, int(n.value)), result


class _InputSlot:
    """One set of batch buffers: pinned host staging, device inputs, copy/consume events, its captured graph."""

    def __init__(self, x_shape, augment):
        b = x_shape[0]
        self.y_pin = PinnedArray((b,))
        self.y_dev = Tensor((b,), Buffer(b, F32))
        self.offs_pin = self.offs_dev = None
        if augment is None:
            self.x_pin = PinnedArray(x_shape)
            self.x_dev = Tensor(x_shape, Buffer(int(np.prod(x_shape)), F32))
        else:
            # raw uint8 images (held in a 4-byte-word buffer), per-image crop offsets / flip bits (int32)
            nbytes = int(np.prod(x_shape))
            self.x_pin = PinnedArray(x_shape, np.uint8)
            self.x_dev = Tensor(((nbytes + 3) // 4,), Buffer((nbytes + 3) // 4, F32))
            self.offs_pin = PinnedArray((b, 3), np.int32)
            self.offs_dev = Tensor((b * 3,), Buffer(b * 3, F32))
        for t in (self.x_dev, self.y_dev):
            t.refs = 1  # external hold: the traversal never returns these to the pool
        self.y_dev.host_src = self.y_pin.array
        lib = _lib.lib()
        evs = []
        for _ in range(2):
            ev = C.c_void_p()
            check(lib.nsk_event_create(0, C.byref(ev)))
            evs.append(ev.value)
        self.copied, self.consumed = evs  # H2D from the pinned buffers done / last step reading x_dev done
        self.copy_pending = False
        self.graph: StepGraph | None = None
        self.loss_slot: int | None = None


class Trainer:
    """Classification training loop over a tape-recorded model.

    ``optimizer`` is ``("sgd", lr, momentum)`` or ``("adamw", Hyperparams, clip_norm|None)``.
    ``augment=(pad, mean, std)``: the inputs are uint8 NHWC images [B, H, W, C]; each step crops (zero pad
    ``pad``), flips and normalises them on the GPU (K18) with host-drawn (dy, dx, flip) per image, and the
    model runs on the NHWC bf16 result (``model.forward(x_nhwc=...)``).
    """

    def __init__(self, session, model, x_shape, classes: int, optimizer=("sgd", 0.1, 0.9), graph: bool = True,
                 warmup: int = 2, dp=None, augment=None, augment_seed: int = 0):
        self.s = session
        self.model = model
        self.classes = classes
        self.opt = optimizer
        self.use_graph = graph
        self.warmup = warmup
        self.dp = dp
        self.x_shape = tuple(x_shape)
        b = self.x_shape[0]
        self.augment = augment
        self._slots = [_InputSlot(self.x_shape, augment)]
        self._cur = 0  # input slot the next step reads
        self._async_n = 0
        self._copy_stream = None
        if augment is not None:
            pad, mean, std = augment
            c = self.x_shape[3]
            self.aug_stats = Tensor((2, c), Buffer(2 * c, F32))
            self.aug_stats.buffer.upload(np.stack([np.broadcast_to(np.asarray(mean, np.float32), (c,)),
                                                   np.broadcast_to(np.asarray(std, np.float32), (c,))]))
            self.aug_rng = np.random.default_rng(augment_seed)
        # token models: ids are validated on the host at staging time (sync-free inside the step)
        self.input_classes = getattr(model, "input_classes", None)
        if self.input_classes is not None:
            self.x_dev.host_src = self.x_pin.array
        self.steps_done = 0
        self.fresh_at_capture = None

    # the current input slot's buffers (slot 0 unless step_async alternates)
    x_pin = property(lambda self: self._slots[self._cur].x_pin)
    y_pin = property(lambda self: self._slots[self._cur].y_pin)
    x_dev = property(lambda self: self._slots[self._cur].x_dev)
    y_dev = property(lambda self: self._slots[self._cur].y_dev)
    offs_pin = property(lambda self: self._slots[self._cur].offs_pin)
    offs_dev = property(lambda self: self._slots[self._cur].offs_dev)
    graph = property(lambda self: self._slots[self._cur].graph)
    loss_slot = property(lambda self: self._slots[self._cur].loss_slot)

    # -- the step body (recorded on the tape) --
    def _body(self) -> DeviceScalar:
        s = self.s
        if self.dp is not None:
            self.dp.begin_step()
        y = data_from_device(self.y_dev)
        if self.augment is None:
            logits = self.model.forward(data_from_device(self.x_dev))
        else:
            from .tensor import empty_tensor

            b, h, w, c = self.x_shape
            xa = empty_tensor(s.pool, (b, h, w, c), BF16)
            check(_lib.lib().nsk_augment_crop_flip(self.x_dev.ptr, self.offs_dev.ptr, xa.ptr, b, h, w, c,
                                                   int(self.augment[0]), self.aug_stats.ptr,
                                                   self.aug_stats.ptr + 4 * c, c, _lib.stream()))
            logits = self.model.forward(x_nhwc=data_from_device(xa))
        loss = nn.cross_entropy(logits, y, s.pool)
        s.push_named("train.loss", loss)
        backward(s.tape(), s.grad_cache, s.pool)
        if self.dp is not None:
            self.dp.finish_backward()
        kind = self.opt[0]
        if kind == "sgd":
            nn.sgd_step(s.param_group, s.grad_cache, self.opt[1], self.opt[2])
        elif kind == "adamw":
            hp, clip = self.opt[1], self.opt[2]
            if self.dp is not None:  # average before the norm is taken (clip sees the global gradient)
                nn.scale_grads(s.grad_cache, s.param_group.scale_dev())
            if clip is not None:
                nn.clip_grad_norm(s.grad_cache, clip)
            nn.adamw_step(s.param_group, s.grad_cache, hp, apply_group_scale=False)
        else:
            raise NskRuntimeError(f"unknown optimizer {kind!r}")
        s.grad_cache.zero_after_step()
        if loss._scalar is None:
            raise NskRuntimeError("loss was not reclaimed by backward()")
        return loss._scalar

    def stage(self, x_host, y_host, offsets=None) -> None:
        """Host batch -> pinned -> device (async on the compute stream). With ``augment``, ``offsets`` [B, 3]
        (dy, dx, flip) default to a draw from the trainer's Generator (oracle/restated.draw_crop_flip order)."""
        y = np.asarray(y_host, dtype=np.float32).reshape(-1)
        check_index_values(y, self.classes, "target")
        if self.input_classes is not None:
            check_index_values(np.asarray(x_host, dtype=np.float32), self.input_classes, "onehot")
        lib = _lib.lib()
        sl = self._slots[self._cur]
        st = self._copy_stream if self._copy_stream is not None else _lib.stream()
        if sl.copy_pending:
            check(lib.nsk_event_sync(sl.copied))  # the previous H2D finished reading the pinned buffers
        if st != _lib.stream():
            check(lib.nsk_event_wait(st, sl.consumed))  # the last step reading this slot's device inputs is done
        np.copyto(self.x_pin.array, np.asarray(x_host, dtype=self.x_pin.dtype).reshape(self.x_shape))
        np.copyto(self.y_pin.array, y)
        check(lib.nsk_memcpy_h2d(self.x_dev.ptr, self.x_pin.ptr, self.x_pin.nbytes, st))
        if self.augment is not None:
            from .data import _draw_crop_flip

            offs = _draw_crop_flip(self.aug_rng, self.x_shape[0], int(self.augment[0])) if offsets is None \
                else np.asarray(offsets, np.int32)
            np.copyto(self.offs_pin.array, offs.reshape(-1, 3))
            check(lib.nsk_memcpy_h2d(self.offs_dev.ptr, self.offs_pin.ptr, self.offs_pin.nbytes, st))
        check(lib.nsk_memcpy_h2d(self.y_dev.ptr, self.y_pin.ptr, self.y_pin.nbytes, st))
        check(lib.nsk_event_record(sl.copied, st))
        sl.copy_pending = True
        if st != _lib.stream():
            check(lib.nsk_event_wait(_lib.stream(), sl.copied))  # compute waits for the copy, not the host

    def run_staged(self) -> DeviceScalar:
        """One step on the already-staged device batch (no host copies)."""
        sl = self._slots[self._cur]
        if sl.graph is not None:
            sl.graph.launch()
            self.s.param_group.step_count += 1  # the replayed optimizer step (recording counted the captured one)
            sc = DeviceScalar(sl.loss_slot)
        elif self.use_graph and self.steps_done >= self.warmup:
            fresh = self.s.pool.stats()["fresh"]
            sl.graph, sc = capture(self._body)
            if self.s.pool.stats()["fresh"] != fresh:
                raise NskRuntimeError("pool was not warm at capture time")
            sl.loss_slot = sc.slot
            sl.graph.launch()
            sc = DeviceScalar(sl.loss_slot)
        else:
            sc = self._body()
        check(_lib.lib().nsk_event_record(sl.consumed, _lib.stream()))
        self.steps_done += 1
        return sc

    def step(self, x_host, y_host, offsets=None) -> DeviceScalar:
        """The public call: copy the host batch in, run one training step, return the loss (on device)."""
        self.stage(x_host, y_host, offsets)
        # the pinned staging buffers may be overwritten by the next stage() only after this step's copies ran
        return self.run_staged()

    def evaluate(self, x_host, y_host) -> tuple[float, int]:
        """Inference pass (§8(f) 4): forward with BatchNorm in eval mode (running statistics), the loss and the
        argmax-correct count; nothing is kept for backward (tape_clear, autodiff.py:83-95). uint8 augment
        inputs are normalised without crop or flip (centre offsets)."""
        from .builtins import accuracy_count
        from .tensor import empty_tensor

        s, lib, st = self.s, _lib.lib(), _lib.stream()
        y = autodiff.make_data(s.pool, np.asarray(y_host, np.float32).reshape(-1))
        if self.augment is None:
            logits = self.model.forward(autodiff.make_data(s.pool, np.asarray(x_host, np.float32)), train=False)
        else:
            imgs = np.ascontiguousarray(x_host, dtype=np.uint8)
            b, h, w, c = imgs.shape
            raw = Buffer((imgs.size + 3) // 4, F32)
            raw.upload(np.frombuffer(imgs.tobytes() + b"\0" * (-imgs.size % 4), np.float32))
            pad = int(self.augment[0])
            offs = Buffer(b * 3, F32)
            offs.upload(np.tile(np.array([pad, pad, 0], np.int32), b).view(np.float32))
            xa = empty_tensor(s.pool, (b, h, w, c), BF16)
            check(lib.nsk_augment_crop_flip(raw.ptr, offs.ptr, xa.ptr, b, h, w, c, pad, self.aug_stats.ptr,
                                            self.aug_stats.ptr + 4 * c, c, st))
            logits = self.model.forward(x_nhwc=data_from_device(xa), train=False)
        loss = nn.cross_entropy(logits, y, s.pool)
        correct = accuracy_count(logits, y)
        value = float(loss.item())
        s.push_named("eval.loss", loss)
        s.tape().clear(s.pool)
        return value, int(correct)

    def step_async(self, x_host, y_host, offsets=None) -> DeviceScalar:
        """``step`` with the host->device copy on a copy stream into one of two input slots, so the copy (and
        the host-side staging) of batch i+1 overlaps the device work of batch i. Each slot has its own
        captured graph; the returned loss is still a device scalar (read it when needed)."""
        if len(self._slots) < 2:
            self._slots.append(_InputSlot(self.x_shape, self.augment))
            if self.input_classes is not None:  # token ids validated on the host at staging (as for slot 0)
                self._slots[1].x_dev.host_src = self._slots[1].x_pin.array
            s = C.c_void_p()
            check(_lib.lib().nsk_stream_create(C.byref(s)))
            self._copy_stream = s.value
        self._cur = self._async_n % 2
        self._async_n += 1
        self.stage(x_host, y_host, offsets)
        return self.run_staged()

    @property
    def launches_per_step(self) -> int:
        g = self._slots[0].graph
        return g.nodes if g is not None else -1
