"""Data-parallel training: one process per GPU, bucketed NCCL all-reduce overlapped with backward.

The reference has no distributed path. The exchange step of
data parallelism is the gradient sum, and the reference's traversal already
exposes the moment a parameter's gradient is final: the param-fire branch of
``_fire`` (autodiff.py:394-399). ``GradCache.hooks`` runs there; this module
counts finished parameters per bucket of the flat gradient arena (laid out in
reverse declaration order, the order backward finishes them) and, as soon as
a bucket is complete, launches its in-place ``ncclAllReduce`` on a separate
comm stream after an event on the compute stream -- the transfer overlaps the
rest of backward. The optimizer waits on the comm stream and folds the 1/N
average into its update (ParamGroup.grad_scale), so averaging costs no pass.

Rendezvous: rank 0's ncclUniqueId travels over torch.distributed (gloo, host
only); the collectives themselves are libnskb's NCCL calls over NVLink 5 /
NVSwitch.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .side import SIDE
from ._lib import F32, check
from .errors import NskRuntimeError


def _event():
    ev = C.c_void_p()
    check(_lib.lib().nsk_event_create(0, C.byref(ev)))
    return ev.value


class DataParallel:
    """``allreduce`` (tests only): a callable ``(ptr, count, dtype, stream)`` used instead of NCCL -- e.g. a host
    gloo all-reduce so two processes sharing one GPU can exercise the bucketing and hooks; no NCCL communicator
    is created then."""

    def __init__(self, session, rank: int, world: int, bucket_mb: float = 4.0, uid: bytes | None = None,
                 allreduce=None):
        self.s = session
        self.rank, self.world = rank, world
        self.bucket_elems = max(1, int(bucket_mb * (1 << 20) / 4))
        lib = _lib.lib()
        self.comm = None
        self._allreduce_fn = allreduce
        if allreduce is None:
            if uid is None:
                uid = self._exchange_uid()
            buf = (C.c_uint8 * 128).from_buffer_copy(uid)
            comm = C.c_void_p()
            check(lib.nsk_comm_init(rank, world, buf, C.byref(comm)))
            self.comm = comm.value
        self.launch_log: list[int] = []  # bucket indices in launch order (host-side record, for tests)
        s = C.c_void_p()
        check(lib.nsk_stream_create(C.byref(s)))
        self.comm_stream = s.value
        self.buckets = None  # list of (start, count, names)
        self.pending = None
        self.launched = None
        self.ev_compute = []
        self.ev_done = _event()
        session.param_group.grad_scale = 1.0 / world
        session.grad_cache.hooks.append(self._on_param_final)

    def allreduce(self, ptr: int, count: int, dtype: int, stream) -> None:
        """In-place sum over ranks of ``count`` elements at ``ptr``, enqueued on ``stream``."""
        if self._allreduce_fn is not None:
            self._allreduce_fn(ptr, count, dtype, stream)
        else:
            check(_lib.lib().nsk_allreduce(self.comm, ptr, count, dtype, stream))

    def _exchange_uid(self) -> bytes:
        import torch.distributed as dist

        if not dist.is_initialized():
            dist.init_process_group(backend="gloo")
        obj = [None]
        if self.rank == 0:
            raw = (C.c_uint8 * 128)()
            check(_lib.lib().nsk_comm_unique_id(raw))
            obj = [bytes(raw)]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    # -- parameter sync (guard: init is already bit-identical by seed) --
    def broadcast_params(self):
        """Rank 0's parameters to everyone: all-reduce of (rank==0 ? w : 0)."""
        lib, st = _lib.lib(), _lib.stream()
        for _name, t in self.s.param_group.params:
            if self.rank != 0:
                check(lib.nsk_fill_f32(t.ptr, t.numel, 0.0, st))
            self.allreduce(t.ptr, t.numel, F32, st)
            t.version += 1
        _lib.sync()

    def _build_buckets(self):
        cache = self.s.grad_cache
        offs = cache.offsets
        order = sorted(offs.items(), key=lambda kv: kv[1])
        buckets, cur, start = [], [], 0
        end = 0
        for name, off in order:
            if not cur:
                start = off
            cur.append(name)
            end = off + cache.grads[name].capacity
            if end - start >= self.bucket_elems:
                buckets.append((start, end - start, cur))
                cur = []
        if cur:
            buckets.append((start, cache.arena.capacity - start, cur))
        else:
            last = buckets[-1]
            buckets[-1] = (last[0], cache.arena.capacity - last[0], last[2])
        self.buckets = buckets
        self.owner = {n: i for i, (_s, _c, names) in enumerate(buckets) for n in names}
        self.ev_compute = [_event() for _ in buckets]

    def _on_param_final(self, name: str):
        if self.buckets is None:
            return
        i = self.owner.get(name)
        if i is None:
            return
        self.pending[i] -= 1
        if self.pending[i] == 0:
            self._launch(i)

    def _launch(self, i):
        lib = _lib.lib()
        start, count, _names = self.buckets[i]
        ptr = self.s.grad_cache.arena.ptr + 4 * start
        check(lib.nsk_event_record(self.ev_compute[i], _lib.stream()))
        check(lib.nsk_event_wait(self.comm_stream, self.ev_compute[i]))
        SIDE.order_after(self.comm_stream)  # weight gradients forked onto the side stream (side.py)
        self.allreduce(ptr, count, F32, self.comm_stream)
        self.launched[i] = True
        self.launch_log.append(i)

    def begin_step(self):
        if self.buckets is None and self.s.grad_cache.arena is not None:
            self._build_buckets()
        if self.buckets is not None:
            self.pending = [len(names) for (_s, _c, names) in self.buckets]
            self.launched = [False] * len(self.buckets)

    def finish_backward(self):
        """Join the comm stream before the optimizer reads the gradients."""
        lib, st = _lib.lib(), _lib.stream()
        cache = self.s.grad_cache
        if self.buckets is None:
            # first (eager) step: the arena does not exist yet -> reduce parameter by parameter
            SIDE.order_after(st)
            for name, buf in cache.grads.items():
                self.allreduce(buf.ptr, buf.capacity, F32, st)
            return
        for i, done in enumerate(self.launched):
            if not done:
                self._launch(i)
        check(lib.nsk_event_record(self.ev_done, self.comm_stream))
        check(lib.nsk_event_wait(st, self.ev_done))
        self.pending = None

    def allreduce_count(self, value: int) -> int:
        """Sum of an integer over ranks (e.g. correct predictions for accuracy, bit-exact)."""
        from .tensor import Buffer

        if self.comm is None:  # injected transport (tests): the host process group sums it
            import torch
            import torch.distributed as dist

            t = torch.tensor([int(value)], dtype=torch.int64)
            dist.all_reduce(t)
            return int(t[0])
        b = Buffer(1, F32)
        arr = np.array([value], np.int32)
        lib, st = _lib.lib(), _lib.stream()
        check(lib.nsk_memcpy_h2d(b.ptr, arr.ctypes.data, 4, st))
        check(lib.nsk_allreduce_i32(self.comm, b.ptr, 1, st))
        check(lib.nsk_memcpy_d2h(arr.ctypes.data, b.ptr, 4, st))
        _lib.sync()
        return int(arr[0])
