"""Accuracy study on the GPU (the reference's ``accuracy`` command,
zk/cli.py:98-130,329-354), with a double-double GPU reference in place of
the exact big-integer oracle.

The reference scores each method against ``oracle_table`` evaluated at the
EXACT rationals i/(P-1) (zk/cli.py:117-121) while the candidates see their
binary64 roundings. Here the reference values come from
``zk_radial_eval_dd``: the Jacobi recursion in double-double at the
double-double points i/(P-1) (hi = binary64 rounding, lo = exact residual),
rounded once -- equal to the correctly rounded exact value except at
near-ties, and seconds instead of minutes at n = 200.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

import numpy as np

from . import _lib
from .baselines import radial_direct_table, radial_ztt_table
from .evaluate import basis_matrix
from .modes import Mode, as_mode_set, mode_arrays
from .tables import linear_radial_grid

METHODS = ("jacobi", "direct", "ztt")  # zk/cli.py:27
MAX_ACCURACY_N = 150  # zk/cli.py:40 (kept for CLI compatibility)
ACCURACY_HEADER = ("n", "m", "k", "method", "max_abs_err")  # zk/cli.py:28


@dataclass(frozen=True)
class AccuracyRow:
    """zk/cli.py:49-55."""

    n: int
    m: int
    deriv_order: int
    method: str
    max_abs_err: float


def rational_grid_dd(num_points: int) -> tuple[np.ndarray, np.ndarray]:
    """(hi, lo) with hi + lo = i/(P-1) to ~106 bits; hi = linear_radial_grid(P)."""
    hi = linear_radial_grid(num_points)
    q = num_points - 1
    lo = np.array([float(Fraction(i, q) - Fraction(float(h))) for i, h in enumerate(hi)])
    return hi, lo


def reference_table(modes, rho_hi, rho_lo=None, deriv_order: int = 0) -> np.ndarray:
    """(P, M) double-double reference values at rho_hi + rho_lo, rounded once."""
    ms = as_mode_set(modes)
    hi = np.ascontiguousarray(rho_hi, dtype=np.float64)
    lo = None if rho_lo is None else np.ascontiguousarray(rho_lo, dtype=np.float64)
    P, M = hi.size, len(ms)
    out = np.empty((P, M), dtype=np.float64, order="F")
    if P and M:
        n, m = mode_arrays(ms)
        ctx = _lib.context()
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_radial_eval_dd(
            ctx.handle, plan.handle, _lib.dptr(hi), _lib.dptr(lo) if lo is not None else None, P,
            int(deriv_order), _lib.dptr(out), P, _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT),
            "zk_radial_eval_dd")
    return out


def _sweep_modes(n_max: int):
    """All (n, m >= 0) modes with n <= n_max (zk/cli.py:70-74)."""
    return tuple(Mode(n, m) for n in range(n_max + 1) for m in range(n % 2, n + 1, 2))


def run_accuracy(n_max: int, methods: Sequence[str] = METHODS, grid_size: int = 100,
                 k_max: int = 0, serial: bool = False) -> list[AccuracyRow]:
    """zk/cli.py:98-130 on the GPU: max-abs error of each method per (n, m, k)."""
    if n_max < 0 or n_max > MAX_ACCURACY_N:
        raise ValueError(f"n_max must be in 0..{MAX_ACCURACY_N}, got {n_max}")
    for method in methods:
        if method not in METHODS:
            raise ValueError(f"unknown method {method!r}")
    modes = _sweep_modes(n_max)
    hi, lo = rational_grid_dd(grid_size)
    n_arr, m_arr = mode_arrays(modes)
    rows: list[AccuracyRow] = []
    for k in range(k_max + 1):
        ref = reference_table(modes, hi, lo, k)
        for method in methods:
            if method == "ztt" and k:
                continue
            if method == "jacobi":
                cand = basis_matrix(n_arr, m_arr, hi, k)
            elif method == "direct":
                cand = radial_direct_table(modes, hi, k)
            else:
                cand = radial_ztt_table(modes, hi)
            errs = np.max(np.abs(cand - ref), axis=0)
            rows.extend(AccuracyRow(md.n, md.m, k, method, float(e)) for md, e in zip(modes, errs))
    order = {m: i for i, m in enumerate(methods)}
    rows.sort(key=lambda r: (r.n, r.m, r.deriv_order, order[r.method]))
    return rows
