"""The reference's float baselines on the GPU.

``radial_direct`` (zk/evaluate.py:189-208) -- the alternating power sum with
exact integer coefficients rounded once to binary64 -- and the Zernike
three-term recursion ``radial_ztt_table`` / ``radial_ztt``
(zk/evaluate.py:211-247). They are the paper's comparison baselines for the
stability study (the direct sum is useless by n ~ 60, README of the
reference); the production path is the Jacobi recursion (``evaluate.py``).
Same names, arguments and validation as the reference; values from
``csrc/zk_baselines.cu`` through the C ABI.
"""

from __future__ import annotations

from math import comb

import numpy as np

from . import _lib
from .evaluate import _radial_mode
from .modes import as_mode_set, mode_arrays
from .tables import radial_grid

_HOST = _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT


def radial_terms(n: int, m_abs: int, deriv_order: int = 0) -> list[tuple[int, int]]:
    """(exponent, exact integer coefficient) in descending exponent order of
    R_n^|m| or its deriv_order-th derivative: coefficient of rho^(n-2s) is
    (-1)^s C(n-s, s) C(n-2s, (n-|m|)/2 - s) (zk/exact.py:48-80 semantics)."""
    j = (n - m_abs) // 2
    terms = [(n - 2 * s, (-1) ** s * comb(n - s, s) * comb(n - 2 * s, j - s))
             for s in range(j + 1)]
    if deriv_order not in (0, 1, 2, 3):
        raise ValueError(f"derivative order must be 1..3, got {deriv_order}")
    for _ in range(deriv_order):
        terms = [(e - 1, c * e) for e, c in terms if e >= 1]
    return terms


def radial_direct_table(modes, grid, deriv_order: int = 0) -> np.ndarray:
    """Direct-sum values for a mode list, (P, M) F-ordered."""
    ms = as_mode_set(modes)
    rho = np.ascontiguousarray(radial_grid(grid))
    coef, ptr, low = [], [0], []
    for md in ms:
        terms = radial_terms(md.n, md.m_abs, deriv_order)
        coef.extend(float(c) for _, c in terms)  # exact int -> correctly rounded binary64
        ptr.append(len(coef))
        low.append(terms[-1][0] if terms else 0)
    P, M = rho.size, len(ms)
    out = np.empty((P, M), dtype=np.float64, order="F")
    if P and M:
        c = np.ascontiguousarray(coef if coef else [0.0], dtype=np.float64)
        pt = np.ascontiguousarray(ptr, dtype=np.int32)
        lo = np.ascontiguousarray(low, dtype=np.int32)
        ctx = _lib.context()
        _lib.check(_lib.lib.zk_direct_eval(ctx.handle, _lib.dptr(rho), P, _lib.dptr(c),
                                           _lib.dptr(pt), _lib.dptr(lo), M, _lib.dptr(out), P,
                                           _HOST), "zk_direct_eval")
    return out


def radial_direct(n: int, m_abs: int, grid, deriv_order: int = 0) -> np.ndarray:
    """zk/evaluate.py:189-208 (unstable baseline, kept deliberately)."""
    mode = _radial_mode(n, m_abs)
    radial_grid(grid)
    return radial_direct_table((mode,), grid, deriv_order)[:, 0].copy()


def radial_ztt_table(modes, grid) -> np.ndarray:
    """zk/evaluate.py:211-241: Zernike three-term recursion, (P, M), value only."""
    ms = as_mode_set(modes)
    rho = np.ascontiguousarray(radial_grid(grid))
    P, M = rho.size, len(ms)
    out = np.empty((P, M), dtype=np.float64, order="F")
    if P and M:
        n, m = mode_arrays(ms)
        ctx = _lib.context()
        _lib.check(_lib.lib.zk_ztt_eval(ctx.handle, _lib.dptr(rho), P, _lib.dptr(n),
                                        _lib.dptr(m), M, _lib.dptr(out), P, _HOST),
                   "zk_ztt_eval")
    return out


def radial_ztt(n: int, m_abs: int, grid) -> np.ndarray:
    """zk/evaluate.py:244-247 (single mode)."""
    mode = _radial_mode(n, m_abs)
    return radial_ztt_table((mode,), grid)[:, 0].copy()
