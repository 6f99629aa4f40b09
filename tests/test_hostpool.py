"""Host result pool (paper_2409_19156_b200/hostpool.py): recycled buffers for
large numpy results; CPU-only."""

import gc

import numpy as np

from paper_2409_19156_b200 import hostpool


def test_released_buffer_is_reused_only_after_every_view_dies():
    pool = hostpool.ResultPool(1 << 30)
    a = pool.take(3_000_000)
    ptr = a.ctypes.data
    view = a.reshape((1000, 3000), order="F")[:, 5:]
    del a
    gc.collect()
    assert pool.held == 0  # the view still holds the lease
    b = pool.take(3_000_000)
    assert b.ctypes.data != ptr
    del view, b
    gc.collect()
    assert pool.held == 2 * 24_000_000
    c = pool.take(3_000_000)
    assert c.ctypes.data in {ptr} or pool.held == 24_000_000
    c[:] = 1.0  # writable
    assert c.flags.writeable and c.dtype == np.float64 and c.shape == (3_000_000,)


def test_cap_evicts_and_small_arrays_bypass():
    pool = hostpool.ResultPool(40 << 20)
    x, y = pool.take(3_000_000), pool.take(4_000_000)  # 24 MB + 32 MB
    del x, y
    gc.collect()
    assert pool.held <= 40 << 20
    small = pool.take(1000)
    assert small.base is None
    off = hostpool.ResultPool(0)
    assert off.take(3_000_000).base is None
