"""Input pipeline: the reference dataset + prefetch semantics feeding pinned staging and the GPU.

Reference (pkg/src/nsk/):
  dataset.reset_epoch / batch_rows / next_batch   dataset.py:93-142  (seeded per-epoch permutation from a
                                                  Generator created once, contiguous batches, partial last
                                                  batch kept, END_OF_DATA after the last batch)
  concurrency.PrefetchQueue / prefetch_start / prefetch_next   concurrency.py:108-191  (W workers claim batch
                                                  indices in order, bounded queue of capacity 2W, results
                                                  unordered for W > 1, sticky end marker, worker errors
                                                  poison the queue)

B200 restatement: the workers do not build numpy batches that are copied again later -- each claims a slot of
a ring of page-locked host buffers, gathers its batch's rows straight into it (the gather releases the GIL),
and hands the slot to the consumer. The consumer (``DeviceLoader.next``) issues the host->device copy on a
dedicated copy stream, records an event and makes the compute stream wait on it, so the copy of batch i+1
overlaps the training step of batch i. A slot returns to the workers only after its copy has completed.

uint8 image datasets are augmented on the GPU (K18, ``nsk_augment_crop_flip``): pad-4 random crop + horizontal
flip + normalisation, with the crop offsets and flip bits drawn on the host from a Generator seeded by
(seed, epoch, batch index) -- bit-identical to the oracle's draw (oracle/restated.draw_crop_flip) whatever
order the workers finish in.
"""

from __future__ import annotations

import ctypes as C
import os
import queue
import threading

import numpy as np

from . import _lib
from ._lib import check
from .errors import NskRuntimeError


class _EndOfData:
    def __repr__(self):
        return "END_OF_DATA"


END_OF_DATA = _EndOfData()


class _Poison:
    def __init__(self, error: BaseException):
        self.error = error


class PinnedSlot:
    """One ring slot: page-locked host arrays for a batch and the event of its last host->device copy."""

    def __init__(self, x_shape, x_dtype, batch: int, with_offsets: bool):
        lib = _lib.lib()
        self.arrays = {}
        self._ptrs = []
        for name, shape, dt in (("x", x_shape, x_dtype), ("y", (batch,), np.float32),
                                ("offs", (batch, 3), np.int32)):
            if name == "offs" and not with_offsets:
                continue
            nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
            p = C.c_void_p()
            check(lib.nsk_pinned_alloc(max(nbytes, 1), C.byref(p)))
            self._ptrs.append(p.value)
            raw = (C.c_char * max(nbytes, 1)).from_address(p.value)
            self.arrays[name] = np.frombuffer(raw, dtype=dt, count=int(np.prod(shape))).reshape(shape)
        ev = C.c_void_p()
        check(lib.nsk_event_create(0, C.byref(ev)))
        self.event = ev.value
        self.copied = False  # an H2D from this slot is in flight or done (event recorded)
        self.index = -1
        self.rows = 0

    def ptr(self, name: str) -> int:
        return self.arrays[name].ctypes.data

    def wait_copied(self) -> None:
        if self.copied:
            check(_lib.lib().nsk_event_sync(self.event))  # ctypes drops the GIL while waiting
            self.copied = False

    def __del__(self):
        try:
            if _lib._lib is not None:
                for p in self._ptrs:
                    _lib._lib.nsk_pinned_free(p)
                _lib._lib.nsk_event_destroy(self.event)
        except Exception:
            pass


class ImageDataset:
    """In-memory dataset with the reference's epoch/batch semantics (dataset.py:93-142).

    ``features``: float32 [N, C, H, W] (NCHW, fed as is) or uint8 [N, H, W, C] images (augmented on the GPU).
    ``labels``: [N] class ids (float32 on the device, like the reference's CSV labels).

    Data parallelism: ``batch_size`` is the GLOBAL batch. Every rank draws the same global
    permutation (same seed, same Generator) and takes rows [rank*B_loc, (rank+1)*B_loc) of each global batch,
    B_loc = batch_size / world, so the union over ranks is bit-identical to the single-process batch.
    """

    def __init__(self, features, labels, batch_size: int, seed: int = 0, shuffle: bool = True, rank: int = 0,
                 world: int = 1):
        self.features = np.ascontiguousarray(features)
        self.labels = np.ascontiguousarray(labels, dtype=np.float32).reshape(-1)
        if len(self.features) != len(self.labels):
            raise NskRuntimeError(f"dataset has {len(self.features)} rows but {len(self.labels)} labels")
        if batch_size < 1:
            raise NskRuntimeError(f"batch size must be at least 1, got {batch_size}")
        if world < 1 or not 0 <= rank < world or batch_size % world:
            raise NskRuntimeError(f"global batch {batch_size} cannot be split over {world} ranks (rank {rank})")
        self.batch_size = batch_size
        self.rank, self.world = rank, world
        self.local_batch = batch_size // world
        self.seed = seed
        self.shuffle = shuffle
        self.num_rows = len(self.labels)
        self.epoch = 0
        self.permutation = None
        self._rng = None
        self.uint8 = self.features.dtype == np.uint8

    def num_batches(self) -> int:
        return (self.num_rows + self.batch_size - 1) // self.batch_size

    def reset_epoch(self) -> None:
        """Fresh permutation from the Generator created once per dataset (dataset.py:93-100)."""
        if self._rng is None:
            self._rng = np.random.default_rng(self.seed)
        self.epoch += 1
        self.permutation = self._rng.permutation(self.num_rows) if self.shuffle else np.arange(self.num_rows)

    def global_rows(self, index: int) -> int:
        """Rows in global batch ``index`` (the last one may be partial, dataset.py:118-121)."""
        lo = index * self.batch_size
        return max(0, min(lo + self.batch_size, self.num_rows) - lo)

    def batch_rows(self, index: int) -> np.ndarray:
        """Row ids of this rank's share of batch ``index`` under the current permutation (dataset.py:114-121):
        the contiguous global batch, then the rank's contiguous slice of it."""
        if self.permutation is None:
            self.reset_epoch()
        lo = index * self.batch_size
        rows = self.permutation[lo:min(lo + self.batch_size, self.num_rows)]
        if self.world == 1:
            return rows
        return rows[self.rank * self.local_batch:(self.rank + 1) * self.local_batch]


    @classmethod
    def from_cifar_bin(cls, paths, batch_size: int, **kw) -> "ImageDataset":
        """A uint8 dataset from CIFAR-10 binary batches (read_cifar_bin)."""
        images, labels = read_cifar_bin(paths)
        return cls(images, labels, batch_size, **kw)


# ---- on-disk image format (the reference reads CSV only, dataset.py:48-90) ----
CIFAR_RECORD = 1 + 3 * 32 * 32  # label byte, then the 1024 red, 1024 green and 1024 blue bytes (row-major 32x32)


def read_cifar_bin(paths) -> tuple[np.ndarray, np.ndarray]:
    """CIFAR-10 binary batches (``data_batch_*.bin`` / ``test_batch.bin``, memory-mapped) -> uint8 images
    [N, 32, 32, 3] (NHWC: the layout the GPU crop/flip/normalise reads) and float32 labels, files concatenated in
    the order given."""
    if isinstance(paths, (str, os.PathLike)):
        paths = [paths]
    images, labels = [], []
    for path in paths:
        raw = np.memmap(path, dtype=np.uint8, mode="r")
        if raw.size == 0 or raw.size % CIFAR_RECORD:
            raise NskRuntimeError(f"{path}: {raw.size} bytes is not a whole number of {CIFAR_RECORD}-byte records")
        rec = raw.reshape(-1, CIFAR_RECORD)
        labels.append(rec[:, 0].astype(np.float32))
        images.append(rec[:, 1:].reshape(-1, 3, 32, 32).transpose(0, 2, 3, 1))
    return np.ascontiguousarray(np.concatenate(images)), np.concatenate(labels)


def write_cifar_bin(path, images: np.ndarray, labels) -> None:
    """The inverse of read_cifar_bin for one file: uint8 NHWC [N, 32, 32, 3] images and labels 0..255."""
    images = np.asarray(images)
    labels = np.asarray(labels)
    if images.dtype != np.uint8 or images.shape[1:] != (32, 32, 3) or len(images) != len(labels):
        raise NskRuntimeError("write_cifar_bin needs uint8 [N, 32, 32, 3] images and N labels")
    if labels.min() < 0 or labels.max() > 255 or np.any(labels != np.round(labels)):
        raise NskRuntimeError("CIFAR labels are single bytes")
    rec = np.empty((len(images), CIFAR_RECORD), np.uint8)
    rec[:, 0] = labels.astype(np.uint8)
    rec[:, 1:] = images.transpose(0, 3, 1, 2).reshape(len(images), -1)
    rec.tofile(path)


def _draw_crop_flip(rng: np.random.Generator, n: int, pad: int) -> np.ndarray:
    """Per image (dy, dx, flip), the order oracle/restated.draw_crop_flip uses."""
    out = np.empty((n, 3), np.int32)
    for i in range(n):
        out[i, 0] = rng.integers(0, 2 * pad + 1)
        out[i, 1] = rng.integers(0, 2 * pad + 1)
        out[i, 2] = rng.integers(0, 2)
    return out


def batch_generator(seed: int, epoch: int, index: int) -> np.random.Generator:
    return np.random.default_rng([seed, epoch, index])


class DeviceLoader:
    """Prefetching loader: W worker threads fill a pinned ring; ``next`` stages a batch on the device.

    ``trainer`` provides the device destination buffers (``Trainer.x_dev``/``y_dev``/``offs_dev``). With
    ``workers == 1`` batches are produced in order on the consumer thread (dataset.py:124-142, no queue).
    """

    def __init__(self, ds: ImageDataset, trainer, workers: int = 3, capacity: int | None = None):
        if workers < 1:
            raise NskRuntimeError(f"prefetch needs at least 1 worker, got {workers}")
        self.ds = ds
        self.tr = trainer
        self.workers = workers
        self.capacity = capacity or 2 * workers
        if self.capacity < 1:
            raise NskRuntimeError(f"prefetch capacity must be at least 1, got {self.capacity}")
        self.pad = int(trainer.augment[0]) if getattr(trainer, "augment", None) is not None else 0
        if ds.uint8 != (getattr(trainer, "augment", None) is not None):
            raise NskRuntimeError("uint8 image datasets need a Trainer built with augment=(pad, mean, std), "
                                  "float32 NCHW datasets one without")
        # labels are validated once here; inside captured steps nothing reads them on the host
        from .tensor import check_index_values

        check_index_values(ds.labels, trainer.classes, "target")
        b = ds.local_batch
        x_shape = (b,) + ds.features.shape[1:]
        self.slots = [PinnedSlot(x_shape, ds.features.dtype, b, ds.uint8) for _ in range(self.capacity + 1)]
        lib = _lib.lib()
        s = C.c_void_p()
        check(lib.nsk_stream_create(C.byref(s)))
        self.copy_stream = s.value
        self._free: queue.Queue = queue.Queue()
        for sl in self.slots:
            self._free.put(sl)
        self._epoch: _Epoch | None = None
        self._threads: list[threading.Thread] = []
        self._cursor = 0

    # -- producers --
    def _fill(self, slot: PinnedSlot, index: int) -> None:
        ds = self.ds
        rows = ds.batch_rows(index)
        n = len(rows)
        slot.wait_copied()  # the previous copy out of this slot has finished
        np.take(ds.features, rows, axis=0, out=slot.arrays["x"][:n])
        np.take(ds.labels, rows, axis=0, out=slot.arrays["y"][:n])
        if ds.uint8:
            offs = _draw_crop_flip(batch_generator(ds.seed, ds.epoch, index), ds.global_rows(index), self.pad)
            slot.arrays["offs"][:n] = offs[ds.rank * ds.local_batch:ds.rank * ds.local_batch + n]
        slot.index, slot.rows = index, n

    def _worker(self, ep: "_Epoch") -> None:
        """One prefetch worker of epoch ``ep`` (concurrency.py:143-160). Everything it touches belongs to its own
        epoch, so a reset_epoch while it runs cannot mix its batches or counters into the next epoch."""
        try:
            while not ep.stop.is_set():
                i = ep.claim(self.ds.num_batches())
                if i is None:
                    break
                slot = self._get_free(ep.stop)
                if slot is None:
                    break
                try:
                    self._fill(slot, i)
                except BaseException as exc:  # noqa: BLE001 - poison the queue (concurrency.py:143-147)
                    self._free.put(slot)
                    ep.put(_Poison(exc))
                    return
                if not ep.put(slot):  # epoch abandoned: the slot goes back to the ring
                    self._free.put(slot)
                    break
        finally:
            if ep.retire():
                ep.put(END_OF_DATA)

    def _get_free(self, stop: threading.Event):
        """A free ring slot, or None once ``stop`` is set (never blocks past a shutdown)."""
        while not stop.is_set():
            try:
                return self._free.get(timeout=0.05)
            except queue.Empty:
                continue
        return None

    def reset_epoch(self) -> None:
        """New epoch (dataset.py:93-112): permutation, then W prefetch workers when W > 1. May be called at any
        point of an epoch: the old epoch's workers are stopped and its staged slots return to the ring."""
        self.shutdown()
        self.ds.reset_epoch()
        self._cursor = 0
        if self.workers > 1:
            ep = _Epoch(self.capacity, self.workers)
            self._epoch = ep
            self._threads = [threading.Thread(target=self._worker, args=(ep,), name=f"nsk-prefetch-{w}",
                                              daemon=True) for w in range(self.workers)]
            for th in self._threads:
                th.start()
        else:
            self._epoch = None

    # -- consumer --
    def _next_slot(self):
        if self.ds.permutation is None:
            self.reset_epoch()
        ep = self._epoch
        if ep is not None:
            item = ep.ready.get()
            if item is END_OF_DATA:
                ep.ready.put(item)  # sticky (concurrency.py:174-177)
                return END_OF_DATA
            if isinstance(item, _Poison):
                ep.stop.set()
                ep.ready.put(item)
                raise item.error
            return item
        if self._cursor >= self.ds.num_batches():
            return END_OF_DATA
        slot = self._free.get()
        self._fill(slot, self._cursor)
        self._cursor += 1
        return slot

    def next(self):
        """Stage the next batch on the device (async): returns its batch index, or END_OF_DATA."""
        slot = self._next_slot()
        if slot is END_OF_DATA:
            return END_OF_DATA
        if slot.rows != self.ds.local_batch:
            self._free.put(slot)
            raise NskRuntimeError("partial final batch: the captured step has a fixed batch shape "
                                  "(drop it or size the dataset to a multiple of the batch)")
        lib, cs = _lib.lib(), self.copy_stream
        tr = self.tr
        # the compute stream's previous reads of the device inputs must finish before they are overwritten
        ev = C.c_void_p()
        check(lib.nsk_event_create(0, C.byref(ev)))
        check(lib.nsk_event_record(ev.value, _lib.stream()))
        check(lib.nsk_event_wait(cs, ev.value))
        check(lib.nsk_memcpy_h2d(tr.x_dev.ptr, slot.ptr("x"), slot.arrays["x"].nbytes, cs))
        check(lib.nsk_memcpy_h2d(tr.y_dev.ptr, slot.ptr("y"), slot.arrays["y"].nbytes, cs))
        if self.ds.uint8:
            check(lib.nsk_memcpy_h2d(tr.offs_dev.ptr, slot.ptr("offs"), slot.arrays["offs"].nbytes, cs))
        check(lib.nsk_event_record(slot.event, cs))
        slot.copied = True
        check(lib.nsk_event_wait(_lib.stream(), slot.event))  # compute waits for the copy, not the host
        check(lib.nsk_event_destroy(ev.value))
        self._free.put(slot)  # refilled only after wait_copied()
        return slot.index

    def shutdown(self) -> None:
        """Stop the current epoch's workers and return every slot they staged (or held) to the ring."""
        ep, self._epoch = self._epoch, None
        if ep is None:
            return
        ep.stop.set()
        for th in self._threads:
            th.join(timeout=5)
        self._threads = []
        while True:
            try:
                item = ep.ready.get_nowait()
            except queue.Empty:
                break
            if item is not END_OF_DATA and not isinstance(item, _Poison):
                self._free.put(item)  # a staged slot


class _Epoch:
    """Per-epoch prefetch state (the reference builds a fresh PrefetchQueue per epoch, dataset.py:103-109):
    the bounded ready queue, the stop flag, the batch-index cursor and the live-worker count."""

    def __init__(self, capacity: int, workers: int):
        self.ready: queue.Queue = queue.Queue(maxsize=capacity)
        self.stop = threading.Event()
        self.lock = threading.Lock()
        self.next_index = 0
        self.active = workers

    def claim(self, num_batches: int) -> int | None:
        with self.lock:
            if self.next_index >= num_batches:
                return None
            i = self.next_index
            self.next_index += 1
            return i

    def put(self, item) -> bool:
        """Enqueue unless the epoch was stopped first (then False: the caller still owns the item)."""
        while not self.stop.is_set():
            try:
                self.ready.put(item, timeout=0.05)
                return True
            except queue.Full:
                continue
        return False

    def retire(self) -> bool:
        """A worker exits; True for the last one of the epoch (it posts END_OF_DATA)."""
        with self.lock:
            self.active -= 1
            return self.active == 0
