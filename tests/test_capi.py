"""C ABI (libzk_b200.so) without a GPU: the library loads, exports every
symbol include/zk_b200.h declares, and its host-side planner reproduces the
reference's integer indexing bit-exactly (golden vectors)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

from paper_2409_19156_b200 import _lib

HEADER = os.path.join(ROOT, "include", "zk_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int64_t|int)\s+(zk_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = header_symbols()
    assert len(names) >= 18
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in names:
        assert hasattr(raw, name), name
    # the ctypes table covers the whole header, nothing more
    assert sorted(_lib.SIGNATURES) == names


def test_version_and_error_string():
    assert _lib.lib.zk_version() >= 10000
    rc = _lib.lib.zk_plan_describe(None, None, -1, None, None, None, None)
    assert rc == _lib.ZK_EINVAL
    assert _lib.lib.zk_last_error()


def _pairs_to_arrays(pairs):
    a = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
    return a[:, 0].copy(), a[:, 1].copy()


def test_planner_matches_reference_dedup(golden):
    for r in range(6):
        n, m = _pairs_to_arrays(golden[f"idx_req{r}"])
        un, um, sc = _lib.describe(n, m)
        keys = golden[f"idx_req{r}_keys"]
        assert np.array_equal(un, keys[:, 0]) and np.array_equal(um, keys[:, 1])
        assert np.array_equal(sc, golden[f"idx_req{r}_scatter"])
        for k in range(4):
            want = golden[f"idx_req{r}_counters"][k].tolist()
            got = list(_lib.step_counters(n, m, k, True)) + list(_lib.step_counters(n, m, k, False))
            assert got == want


@pytest.mark.parametrize("cfg,N", [("c1", 20), ("c2", 100)])
def test_planner_counters_full_sets(golden, cfg, N):
    n, m = _pairs_to_arrays(golden["idx_full200"][: (N + 1) * (N + 2) // 2])
    for k in range(4):
        assert list(_lib.step_counters(n, m, k, True)) == golden[f"{cfg}_k{k}_counter"].tolist()
    un, um, sc = _lib.describe(n, m)
    assert un.size == (N + 2) ** 2 // 4  # U = floor((N+2)^2/4)


def test_planner_rejects_invalid_modes():
    for bad in ([(-1, 0)], [(2, 3)], [(3, 2)], [(4, 2), (5, 2)]):
        n, m = _pairs_to_arrays(bad)
        with pytest.raises(ValueError):
            _lib.describe(n, m)
        with pytest.raises(ValueError):
            _lib.step_counters(n, m, 0, True)


def test_planner_empty_request():
    n = np.zeros(0, np.int32)
    un, um, sc = _lib.describe(n, n)
    assert un.size == 0 and sc.size == 0
    assert _lib.step_counters(n, n, 3, True) == (0, 0)


def test_no_device_fails_loudly():
    count = ctypes.c_int(-1)
    rc = _lib.lib.zk_device_count(ctypes.byref(count))
    if rc == _lib.ZK_OK and count.value > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError):
        _lib.Context(0)


def test_k5_entry_points_validate_without_a_gpu():
    """The K5 (normal-equation allreduce) entry points reject bad arguments
    before touching a device; the packed count is M(M+1)/2 + M."""
    import ctypes as ct
    lib = _lib.lib
    assert lib.zk_gram_packed_count(0) == 0 and lib.zk_gram_packed_count(-3) == 0
    assert lib.zk_gram_packed_count(1891) == 1891 * 1892 // 2 + 1891
    assert lib.zk_gram_pack(None, None, None, 4, None, 0) == _lib.ZK_EINVAL
    assert lib.zk_gram_unpack(None, None, 4, None, None, 0) == _lib.ZK_EINVAL
    arr = ct.c_void_p * 1
    assert lib.zk_gram_allreduce(None, 1, None, None, 4, 0) == _lib.ZK_EINVAL
    assert lib.zk_gram_allreduce(arr(None), 0, arr(None), None, 4, 0) == _lib.ZK_EINVAL
    assert lib.zk_comm_create(None, None, 1, 0, None) == _lib.ZK_EINVAL
    assert lib.zk_comm_info(None, None, None) == _lib.ZK_EINVAL
    assert lib.zk_comm_destroy(None) == _lib.ZK_OK
    assert lib.zk_gram_allreduce_comm(None, None, None, 4, 0) == _lib.ZK_EINVAL
