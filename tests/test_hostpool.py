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


def test_mode_arrays_memoised_per_mode_set():
    """modes.mode_set_entry: one (n, m) walk per mode-set tuple, read-only
    arrays, identity-keyed (an equal but distinct tuple gets its own entry)."""
    from paper_2409_19156_b200 import modes as zm

    ms = zm.full_mode_set(12)
    n1, m1 = zm.mode_arrays(ms)
    n2, m2 = zm.mode_arrays(ms)
    assert n1 is n2 and m1 is m2
    assert not n1.flags.writeable and not m1.flags.writeable
    assert n1.tolist() == [md.n for md in ms] and m1.tolist() == [md.m for md in ms]
    twin = tuple(list(ms))
    assert twin is not ms and zm.mode_arrays(twin)[0] is not n1
    lst = list(ms)  # non-tuples are not memoised
    assert zm.mode_arrays(lst)[0] is not zm.mode_arrays(lst)[0]


def test_pinning_failure_is_silent_without_a_device():
    """A recycled buffer that cannot be page-locked (no GPU here) is used
    unpinned, and is not retried."""
    import torch

    if torch.cuda.is_available():
        import pytest
        pytest.skip("CPU-only check")
    pool = hostpool.ResultPool(1 << 30)
    a = pool.take(200_000)
    del a
    gc.collect()
    b = pool.take(200_000)
    assert list(pool.pinned.values()) == [0]
    b[:] = 2.0
    del b
    gc.collect()
    pool.clear()
    assert not pool.pinned


def test_default_pool_keeps_one_buffer_and_release_frees_it():
    """Default bound (no ZK_RESULT_POOL_MB): the most recently released
    buffer only; release() (package: release_buffers()) empties the pool."""
    pool = hostpool.ResultPool(8192 << 20, max_buffers=1)
    a, b, c = pool.take(3_000_000), pool.take(4_000_000), pool.take(5_000_000)
    del a, b, c
    gc.collect()
    assert pool.count() == 1 and pool.held in (24_000_000, 32_000_000, 40_000_000)
    pool.clear()
    assert pool.count() == 0 and pool.held == 0
    assert hostpool.POOL.max_buffers == 1  # the module default
    import paper_2409_19156_b200 as zb
    keep = hostpool.take(2_000_000)
    del keep
    gc.collect()
    assert hostpool.POOL.count() == 1
    zb.release_buffers()  # no contexts without a GPU: only the pool is emptied
    assert hostpool.POOL.count() == 0 and hostpool.POOL.held == 0
