"""Recycled host buffers for large numpy results.

A fresh ``np.empty`` result is untouched anonymous memory: the first write of
every page faults, and at config 2 (a 4.12 GB basis) those faults cost more
than the whole PCIe transfer (measured on the B200 box: 170 ms per
``evaluate_batch`` into fresh memory, 100 ms into already-touched memory,
72 ms into pinned memory; pinning 4 GB costs 0.35-2.7 s, so it does not pay
per call). Large results are therefore carved from buffers that earlier
results released: an array handed out by :func:`take` keeps its buffer alive
through ``ndarray.base``; when the last view dies the buffer returns to a
size-keyed free list and the next result of that size reuses its
already-faulted pages. Bounds: by default the pool keeps ONE released buffer
(the most recent, at most 8 GB) -- the repeated-request case it exists for,
without surprising a drop-in caller with gigabytes of retained RSS after its
results died; ``ZK_RESULT_POOL_MB=<n>`` keeps any number of buffers up to n
MB in total, ``0`` disables the pool. ``release()`` (``release_buffers()`` at
the package level) frees everything the pool holds.
Values never depend on the pool -- every element of a result is written by
the library before it is returned.

A buffer of at most ``ZK_PIN_MAX_MB`` (default 512; 0 disables) is also
page-locked (``zk_host_register``) the first time it is reused, and stays
locked while the pool or a result holds it: from then on the library DMAs
results straight into it (no pinned bounce buffer, no host-side copy). A
100-point x 5,151-mode ... 1,000-point x 5,151-mode request is the size the
reference CLI's ``bench`` loops over; pinning is paid once per recycled
buffer, never for one-off results, and a buffer is unlocked before the pool
drops it.
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np

MIN_POOLED_BYTES = 64 << 10
PIN_MAX_BYTES = int(os.environ.get("ZK_PIN_MAX_MB", "512")) << 20


class _Lease:
    """Owner of one pooled buffer; numpy's ``base`` chain keeps it alive."""

    __slots__ = ("buf", "pool", "__array_interface__", "__weakref__")

    def __init__(self, buf: np.ndarray, pool: "ResultPool"):
        self.buf = buf
        self.pool = pool
        self.__array_interface__ = buf.__array_interface__

    def __del__(self):
        pool, buf = self.pool, self.buf
        self.buf = None
        if pool is not None and buf is not None:
            try:
                pool.give_back(buf)
            except Exception:  # interpreter shutdown: just let the memory go
                pass


class ResultPool:
    def __init__(self, cap_bytes: int, max_buffers: int | None = None):
        self.cap = cap_bytes
        self.max_buffers = max_buffers  # None: bounded by bytes only
        self.free: OrderedDict[int, list[np.ndarray]] = OrderedDict()
        self.held = 0
        self.lock = threading.RLock()  # re-entrant: a GC-triggered release may run inside take()
        # id(buffer) -> registered address, or 0 when registration failed
        # (no device, a page shared with another registered range): not retried
        self.pinned: dict[int, int] = {}

    def _pin(self, buf: np.ndarray) -> None:
        if buf.nbytes > PIN_MAX_BYTES or id(buf) in self.pinned:
            return
        ptr = buf.ctypes.data
        try:
            from . import _lib
            ok = _lib.lib.zk_host_register(ptr, buf.nbytes) == 0
        except Exception:
            ok = False
        self.pinned[id(buf)] = ptr if ok else 0

    def _unpin(self, buf: np.ndarray) -> None:
        ptr = self.pinned.pop(id(buf), 0)
        if ptr:
            from . import _lib
            _lib.lib.zk_host_unregister(ptr)

    def take(self, count: int) -> np.ndarray:
        """A 1-D float64 array of ``count`` elements (contents undefined)."""
        nbytes = 8 * count
        if self.cap <= 0 or nbytes < MIN_POOLED_BYTES:
            return np.empty(count, dtype=np.float64)
        buf = None
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                buf = lst.pop()
                self.held -= nbytes
                if not lst:
                    del self.free[nbytes]
        if buf is None:
            buf = np.empty(count, dtype=np.float64)
        else:
            self._pin(buf)  # reused: page-lock it once (see module doc)
        return np.asarray(_Lease(buf, self))

    def give_back(self, buf: np.ndarray) -> None:
        nbytes = buf.nbytes
        if nbytes > self.cap:
            self._unpin(buf)
            return
        with self.lock:
            while self.free and (self.held + nbytes > self.cap or (
                    self.max_buffers is not None and self.count() >= self.max_buffers)):
                size, lst = next(iter(self.free.items()))  # least recently released size
                self._unpin(lst.pop())
                self.held -= size
                if not lst:
                    del self.free[size]
            if self.max_buffers == 0:
                self._unpin(buf)
                return
            self.free.setdefault(nbytes, []).append(buf)
            self.free.move_to_end(nbytes)
            self.held += nbytes

    def count(self) -> int:
        return sum(len(v) for v in self.free.values())

    def clear(self) -> None:
        with self.lock:
            for lst in self.free.values():
                for buf in lst:
                    self._unpin(buf)
            self.free.clear()
            self.held = 0


def _default_pool() -> ResultPool:
    mb = os.environ.get("ZK_RESULT_POOL_MB")
    if mb is None:
        return ResultPool(8192 << 20, max_buffers=1)
    return ResultPool(int(mb) << 20)


POOL = _default_pool()


def take(count: int) -> np.ndarray:
    return POOL.take(count)


def release() -> None:
    """Free (and unlock) every buffer the result pool holds."""
    POOL.clear()
