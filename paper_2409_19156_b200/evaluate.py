"""Radial / full Zernike evaluation on the B200 -- the reference's L2 API.

Same names, arguments, validation order and exception types as
zk/evaluate.py; every value comes from the CUDA kernels in ``csrc/`` through
the C ABI (``_lib``). Every radial entry point -- single mode, batch, 2-D --
runs the same kernel and operation order, so the reference's cross-entry-point
bitwise invariants (tests/test_batch.py:108-116, tests/test_evaluate.py:201-211)
hold by construction.
"""

from __future__ import annotations

import numpy as np

from . import _lib, hostpool
from .modes import Mode, make_mode
from .tables import angular_grid, radial_grid

MAX_DERIV_ORDER = 3  # zk/evaluate.py:19

_HOST = _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT


def _check_order(k) -> int:
    if k not in (0, 1, 2, 3):
        raise ValueError(f"derivative order must be 0..{MAX_DERIV_ORDER}, got {k}")
    return int(k)


def _radial_mode(n: int, m_abs: int) -> Mode:
    """zk/evaluate.py:22-25."""
    if m_abs < 0:
        raise ValueError("m_abs must be non-negative")
    return make_mode(n, m_abs)


def jacobi_argument(rho: np.ndarray) -> np.ndarray:
    """u = 1 - 2*rho*rho (zk/evaluate.py:28-33). API helper only: the kernels
    form u on the device with the same expression tree."""
    return 1.0 - 2.0 * rho * rho


def jacobi_recursion_steps(j_max: int) -> int:
    """zk/evaluate.py:79-81."""
    return max(0, j_max - 1)


def jacobi_derivative_scale(j: int, alpha: int, beta: int, order: int) -> float:
    """zk/evaluate.py:84-99 (integer rising product, one division by 2**order);
    the planner bakes the same numbers into the device plan."""
    if order < 0:
        raise ValueError(f"order must be >= 0, got {order}")
    if j < order:
        return 0.0
    prod = 1
    for i in range(1, order + 1):
        prod *= alpha + beta + j + i
    return prod / float(2 ** order)


def jacobi_chain(j_max: int, alpha: int, beta: int, x) -> np.ndarray:
    """zk/evaluate.py:36-76 on the GPU: rows P_0..P_jmax at every x."""
    if j_max < 0:
        raise ValueError(f"chain degree must be >= 0, got {j_max}")
    if alpha < 0 or beta < 0:
        raise ValueError(f"need alpha, beta >= 0, got ({alpha}, {beta})")
    x = np.ascontiguousarray(np.atleast_1d(np.asarray(x, dtype=np.float64)))
    out = np.empty((j_max + 1, x.size), dtype=np.float64)
    if x.size == 0:
        return out
    ctx = _lib.context()
    _lib.check(_lib.lib.zk_jacobi_chain(ctx.handle, _lib.dptr(x), x.size, int(j_max), int(alpha),
                                        int(beta), _lib.dptr(out), x.size, _HOST),
               "zk_jacobi_chain")
    return out


def parallel_devices() -> list[int]:
    """Devices ``parallel=True`` spreads a host-level call over: ZK_DEVICES
    (comma list) if set, else every visible GPU."""
    import ctypes
    import os
    env = os.environ.get("ZK_DEVICES")
    if env:
        return [int(x) for x in env.split(",") if x.strip()]
    cnt = ctypes.c_int(0)
    _lib.check(_lib.lib.zk_device_count(ctypes.byref(cnt)), "zk_device_count")
    return list(range(max(1, cnt.value)))


def basis_matrix(mode_n: np.ndarray, mode_m: np.ndarray, rho: np.ndarray, k: int,
                 theta: np.ndarray | None = None, all_orders: bool = False,
                 device: int | None = None, devices: list[int] | None = None):
    """Run K1 (theta None) or K1+K2 on host arrays; returns the (P, M)
    F-ordered matrix, or a list of k+1 of them when ``all_orders``.
    ``devices``: split the points into contiguous shards, one per listed GPU,
    each written straight into its rows of the shared result (one host thread
    per device; the C ABI releases the GIL). Inputs must already be validated."""
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    P, M = rho.size, int(np.asarray(mode_n).size)
    n_out = k + 1 if (all_orders and k > 0) else 1
    flat = hostpool.take(n_out * P * M)
    mats = [flat[o * P * M:(o + 1) * P * M].reshape((P, M), order="F") for o in range(n_out)]
    if theta is not None:
        theta = np.ascontiguousarray(theta, dtype=np.float64)
    devs = list(devices) if devices else [device]
    if P and M:
        from .sharding import shard_range

        def run(shard: int):
            lo, hi = shard_range(P, len(devs), shard)
            if hi <= lo:
                return
            ctx = _lib.context(devs[shard])
            plan = _lib.plan_for(ctx, mode_n, mode_m)
            base = flat.ctypes.data + 8 * lo
            if theta is None:
                rc = _lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.ctypes.data + 8 * lo,
                                             hi - lo, k, int(n_out > 1), base, P, P * M, _HOST)
                _lib.check(rc, "zk_radial_eval")
            else:
                rc = _lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.ctypes.data + 8 * lo,
                                              theta.ctypes.data + 8 * lo, hi - lo, k,
                                              int(n_out > 1), base, P, P * M, _HOST)
                _lib.check(rc, "zk_zernike_eval")

        if len(devs) == 1:
            run(0)
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(len(devs)) as pool:
                list(pool.map(run, range(len(devs))))
    return mats if all_orders else mats[0]


def radial_jacobi(n: int, m_abs: int, grid, deriv_order: int = 0) -> np.ndarray:
    """zk/evaluate.py:157-186: one radial mode (or its rho-derivative)."""
    mode = _radial_mode(n, m_abs)
    _check_order(deriv_order)
    rho = radial_grid(grid)
    col = basis_matrix(np.array([mode.n], np.int32), np.array([mode.m_abs], np.int32), rho,
                       int(deriv_order))
    return col[:, 0]  # the (P, 1) result is one contiguous column: no copy


def zernike_eval(mode: Mode, grid, angles, deriv_order: int = 0) -> np.ndarray:
    """zk/evaluate.py:259-274: radial x cos(m theta) / sin(|m| theta)."""
    rho = radial_grid(grid)
    theta = angular_grid(angles)
    if rho.size != theta.size:
        raise ValueError(
            f"point-wise grids must match: {rho.size} radial vs {theta.size} angular")
    _radial_mode(mode.n, mode.m_abs)
    _check_order(deriv_order)
    col = basis_matrix(np.array([mode.n], np.int32), np.array([mode.m], np.int32), rho,
                       int(deriv_order), theta=theta)
    return col[:, 0]  # the (P, 1) result is one contiguous column: no copy


def radial_at_zero(n: int, m: int) -> float:
    """zk/evaluate.py:250-256: value at the disc centre (case table)."""
    mode = make_mode(n, m)
    if mode.m != 0:
        return 0.0
    return 1.0 if mode.n % 4 == 0 else -1.0


def zernike_radial(r, l, m, dr: int = 0) -> np.ndarray:
    """ZERNIPAX-style batch call: (P,) radii x M modes (l = n) -> (P, M)."""
    from .modes import as_mode_set, mode_arrays
    modes = as_mode_set(zip(np.atleast_1d(l).tolist(), np.atleast_1d(m).tolist()))
    _check_order(dr)
    rho = radial_grid(r)
    n_arr, m_arr = mode_arrays(modes)
    return basis_matrix(n_arr, m_arr, rho, int(dr))


def zernike_basis(r, theta, l, m, dr: int = 0) -> np.ndarray:
    """2-D basis matrix (P, M): column (l, m) = zernike_eval at every point."""
    from .modes import as_mode_set, mode_arrays
    modes = as_mode_set(zip(np.atleast_1d(l).tolist(), np.atleast_1d(m).tolist()))
    _check_order(dr)
    rho = radial_grid(r)
    th = angular_grid(theta)
    if rho.size != th.size:
        raise ValueError(f"point-wise grids must match: {rho.size} radial vs {th.size} angular")
    n_arr, m_arr = mode_arrays(modes)
    return basis_matrix(n_arr, m_arr, rho, int(dr), theta=th)


__all__ = [
    "MAX_DERIV_ORDER", "jacobi_argument", "jacobi_chain", "jacobi_recursion_steps",
    "jacobi_derivative_scale", "radial_jacobi", "zernike_eval", "radial_at_zero",
    "zernike_radial", "zernike_basis", "basis_matrix",
]

