"""Recycled host buffers for large numpy results.

A fresh ``np.empty`` result is untouched anonymous memory: the first write of
every page faults, and at config 2 (a 4.12 GB basis) those faults cost more
than the whole PCIe transfer (measured on the B200 box: 170 ms per
``evaluate_batch`` into fresh memory, 100 ms into already-touched memory,
72 ms into pinned memory; pinning 4 GB costs 0.35-2.7 s, so it does not pay
per call). Large results are therefore carved from buffers that earlier
results released: an array handed out by :func:`take` keeps its buffer alive
through ``ndarray.base``; when the last view dies the buffer returns to a
size-keyed free list (bounded by ``ZK_RESULT_POOL_MB``, default 8192; 0
disables) and the next result of that size reuses its already-faulted pages.
Values never depend on the pool -- every element of a result is written by
the library before it is returned.
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np

MIN_POOLED_BYTES = 1 << 20


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
    def __init__(self, cap_bytes: int):
        self.cap = cap_bytes
        self.free: OrderedDict[int, list[np.ndarray]] = OrderedDict()
        self.held = 0
        self.lock = threading.RLock()  # re-entrant: a GC-triggered release may run inside take()

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
        return np.asarray(_Lease(buf, self))

    def give_back(self, buf: np.ndarray) -> None:
        nbytes = buf.nbytes
        if nbytes > self.cap:
            return
        with self.lock:
            while self.held + nbytes > self.cap and self.free:
                size, lst = next(iter(self.free.items()))  # least recently released size
                lst.pop()
                self.held -= size
                if not lst:
                    del self.free[size]
            self.free.setdefault(nbytes, []).append(buf)
            self.free.move_to_end(nbytes)
            self.held += nbytes

    def clear(self) -> None:
        with self.lock:
            self.free.clear()
            self.held = 0


POOL = ResultPool(int(os.environ.get("ZK_RESULT_POOL_MB", "8192")) << 20)


def take(count: int) -> np.ndarray:
    return POOL.take(count)
