"""A second stream for the weight gradients of the convolutions.

A conv's weight gradient (wgrad) depends on the saved input and the incoming gradient, and feeds only the
optimizer; the input gradient (dgrad) and everything after it in backward do not wait for it. The conv rule
(layers._r_conv2d) forks the wgrad onto this stream -- an event recorded on the compute stream, waited on here
-- so it overlaps the rest of backward (the BatchNorm passes are memory-bound, the small layers leave SMs idle).
Inside a captured step the fork / join become graph edges.

Lifetime: the buffers a forked wgrad reads must outlive it, so pool releases of those buffers are deferred
until ``join`` (the end of ``autodiff.backward``), which makes the compute stream wait for this stream.
Only wgrads that write straight into a gradient-cache sink are forked (nothing on the compute stream reads
their output before the join); the data-parallel all-reduce orders its comm stream after this one too.
NSK_SIDE_WGRAD=0 keeps everything on the compute stream.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _lib
from ._lib import check


class SideStream:
    def __init__(self):
        self._stream = None
        self._ev_fork = None
        self._ev_join = None
        self.active = False
        self.reads: dict[int, object] = {}  # id(buffer) -> buffer read by in-flight side work
        self.deferred: list = []            # (pool, buffer) releases held until join
        self._main = None                   # compute stream while a forward branch runs here (branch())
        self._ev_branch = None

    @staticmethod
    def enabled() -> bool:
        return os.environ.get("NSK_SIDE_WGRAD", "1") != "0"

    def _init(self):
        if self._stream is None:
            lib = _lib.lib()
            # weight gradients share the GPU with the compute stream: one persistent CTA per SM (umma_gemm.cu)
            check(lib.nsk_wgrad_grid_cap(_lib.ctx.sm_count))
            s, e0, e1 = C.c_void_p(), C.c_void_p(), C.c_void_p()
            check(lib.nsk_stream_create(C.byref(s)))
            check(lib.nsk_event_create(0, C.byref(e0)))
            check(lib.nsk_event_create(0, C.byref(e1)))
            self._stream, self._ev_fork, self._ev_join = s.value, e0.value, e1.value

    def fork(self, *buffers) -> int:
        """Order this stream after everything issued so far on the compute stream; hold `buffers` until join.
        Returns the side stream handle to launch on."""
        self._init()
        lib = _lib.lib()
        check(lib.nsk_event_record(self._ev_fork, _lib.stream()))
        check(lib.nsk_event_wait(self._stream, self._ev_fork))
        for b in buffers:
            if b is not None:
                self.reads[id(b)] = b
        self.active = True
        return self._stream

    def defer(self, pool, buffer) -> bool:
        """Pool.release hook: hold the release of a buffer an in-flight side kernel reads (every release while a
        forward branch is being issued here)."""
        if self._main is not None or (self.active and id(buffer) in self.reads):
            self.deferred.append((pool, buffer))
            return True
        return False

    def order_after(self, stream) -> None:
        """Make `stream` wait for the side work issued so far (e.g. the data-parallel comm stream)."""
        if not self.active:
            return
        lib = _lib.lib()
        check(lib.nsk_event_record(self._ev_join, self._stream))
        check(lib.nsk_event_wait(stream, self._ev_join))

    def join(self) -> None:
        """Compute stream waits for the side stream; deferred releases go back to their pools."""
        if not self.active:
            return
        self.order_after(_lib.stream())
        self.active = False
        self.reads.clear()
        held, self.deferred = self.deferred, []
        for pool, buf in held:
            pool.release(buf)


    # ---- forward branches (independent sub-graphs, e.g. a projection shortcut next to conv1) ----
    def branch_begin(self) -> None:
        """Issue the following ops on this stream (ordered after the compute stream so far) until branch_end."""
        self._init()
        if self._ev_branch is None:
            e = C.c_void_p()
            check(_lib.lib().nsk_event_create(0, C.byref(e)))
            self._ev_branch = e.value
        lib = _lib.lib()
        check(lib.nsk_event_record(self._ev_fork, _lib.stream()))
        check(lib.nsk_event_wait(self._stream, self._ev_fork))
        self._main = _lib.ctx.stream
        _lib.ctx.stream = self._stream

    def branch_end(self) -> None:
        """Back to the compute stream; the branch is joined lazily by branch_join."""
        _lib.ctx.stream = self._main
        self._main = None
        check(_lib.lib().nsk_event_record(self._ev_branch, self._stream))
        self._branch_pending = True

    def branch_join(self) -> None:
        """Compute stream waits for the branch; its deferred releases go back to the pool."""
        if not getattr(self, "_branch_pending", False):
            return
        check(_lib.lib().nsk_event_wait(_lib.stream(), self._ev_branch))
        self._branch_pending = False
        if not self.active:  # no weight-gradient work in flight holds these
            held, self.deferred = self.deferred, []
            for pool, buf in held:
                pool.release(buf)


SIDE = SideStream()
