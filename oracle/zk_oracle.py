"""CPU oracle for the Zernike radial hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``zernkit``
(``/root/reference/pkg/src/zernkit``, abbreviated ``zk/`` below) for the one
path this repository accelerates: fp64 radial Zernike evaluation through the
Jacobi three-term recursion, its batch driver, and the 2-D angular product.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
    baseline / ``--impl reference`` arm may import this module. The product
    path (``paper_2409_19156_b200``) never calls it; there is no CPU
    fallback.
  * Every arithmetic expression keeps the reference's operation order
    (numpy, no FMA), so on the same host this port is bitwise equal to the
    reference. That is pinned by ``tests/golden`` (fixtures produced by the
    real reference, ``tests/golden/make_golden.py``) and by
    ``tests/test_oracle.py``.

Parity status: PINNED (golden vectors from the reference itself).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

MAX_DERIV_ORDER = 3  # zk/evaluate.py:19


# --------------------------------------------------------------------------
# mode indexing (zk/modes.py)
# --------------------------------------------------------------------------

def check_mode(n: int, m: int) -> tuple[int, int]:
    """Mode invariants, zk/modes.py:37-43 (n>=0, |m|<=n, n-|m| even)."""
    n, m = int(n), int(m)
    if n < 0 or abs(m) > n or (n - abs(m)) % 2:
        raise ValueError(f"invalid mode ({n}, {m})")
    return n, m


def full_modes(resolution: int) -> list[tuple[int, int]]:
    """zk/modes.py:79-92: n ascending, m ascending over -n, -n+2, ..., n."""
    return [(n, m) for n in range(resolution + 1) for m in range(-n, n + 1, 2)]


def unique_and_scatter(modes) -> tuple[list[tuple[int, int]], list[int]]:
    """zk/modes.py:108-125: (n,|m|) keys in first-appearance order + scatter."""
    slot_of: dict[tuple[int, int], int] = {}
    keys: list[tuple[int, int]] = []
    scatter: list[int] = []
    for n, m in modes:
        key = (int(n), abs(int(m)))
        if key not in slot_of:
            slot_of[key] = len(keys)
            keys.append(key)
        scatter.append(slot_of[key])
    return keys, scatter


def groups_by_alpha(keys) -> list[tuple[int, list[tuple[int, int]]]]:
    """zk/batch.py:61-66: keys grouped by alpha=|m|, sorted by alpha,
    each entry (slot, jacobi degree) in slot order."""
    out: dict[int, list[tuple[int, int]]] = {}
    for slot, (n, a) in enumerate(keys):
        out.setdefault(a, []).append((slot, (n - a) // 2))
    return sorted(out.items())


def step_counts(keys, k: int, shared: bool) -> tuple[int, int]:
    """zk/batch.py:69-94: (recursion_steps, chain_count)."""
    if shared:
        degrees = [max(j for _, j in e) for _, e in groups_by_alpha(keys)]
    else:
        degrees = [(n - a) // 2 for n, a in keys]
    steps = chains = 0
    for d in degrees:
        for i in range(k + 1):
            if d - i >= 0:
                steps += max(0, d - i - 1)  # zk/evaluate.py:79-81
                chains += 1
    return steps, chains


# --------------------------------------------------------------------------
# fp64 engines (zk/evaluate.py)
# --------------------------------------------------------------------------

def jacobi_argument(rho: np.ndarray) -> np.ndarray:
    """zk/evaluate.py:28-33: u = 1 - (2*rho)*rho."""
    return 1.0 - 2.0 * rho * rho


def jacobi_chain(j_max: int, alpha: int, beta: int, x: np.ndarray) -> np.ndarray:
    """zk/evaluate.py:36-76, same expression trees (row j = P_j^(alpha,beta)(x))."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    rows = np.empty((j_max + 1, x.size), dtype=np.float64)
    rows[0] = 1.0
    if j_max >= 1:
        rows[1] = (alpha + 1) + (alpha + beta + 2) * (x - 1) / 2          # :68
    for j in range(2, j_max + 1):
        c = 2 * j + alpha + beta                                          # :70
        lead = 2 * j * (c - j) * (c - 2)                                  # :71
        mid_x = (c - 1) * c * (c - 2)                                     # :72
        mid_const = (c - 1) * (alpha * alpha - beta * beta)               # :73
        last = 2 * (j + alpha - 1) * (j + beta - 1) * c                   # :74
        rows[j] = ((mid_x * x + mid_const) * rows[j - 1] - last * rows[j - 2]) / lead  # :75
    return rows


def derivative_scale(j: int, alpha: int, beta: int, order: int) -> float:
    """zk/evaluate.py:84-99: rising product / 2**order, 0.0 below order."""
    if j < order:
        return 0.0
    prod = 1
    for i in range(1, order + 1):
        prod *= alpha + beta + j + i
    return prod / float(2 ** order)


def numpy_power(rho: np.ndarray, e: int) -> np.ndarray:
    """``rho ** e`` exactly as the reference evaluates it (numpy's array pow,
    which may be 1 ulp off the correctly rounded power)."""
    return rho ** e


def cr_power(rho: np.ndarray, e: int) -> np.ndarray:
    """Correctly rounded rho**e (exact rational power, rounded once; 0**0 = 1).
    The GPU kernels compute their powers this way (double-double, rounded once),
    so the reference algorithm with ``power=cr_power`` is their bitwise oracle
    at every point, not only where numpy's pow happens to be correctly rounded."""
    return np.array([float(Fraction(float(r)) ** e) for r in np.ravel(rho)]).reshape(np.shape(rho))


def cached_cr_power(grid: np.ndarray):
    """``cr_power`` memoised per exponent for one fixed grid: a big request
    (thousands of keys at the same points) asks for each exponent many times."""
    base = np.atleast_1d(np.asarray(grid, dtype=np.float64))
    fr = [Fraction(float(r)) for r in base]
    cache: dict[int, np.ndarray] = {}

    def power(rho: np.ndarray, e: int) -> np.ndarray:
        if rho is not base and not np.array_equal(rho, base):
            return cr_power(rho, e)
        if e not in cache:
            cache[e] = np.array([float(f ** e) for f in fr], dtype=np.float64)
        return cache[e]

    return power


def assemble(rho: np.ndarray, m: int, j: int, k: int, ch, power=numpy_power) -> np.ndarray:
    """zk/evaluate.py:102-154. ``ch[i]`` = P_{j-i}^{(m+i, i)}(u).

    Expressions are written exactly as numpy evaluates the reference's
    (left-to-right products, python-int prefactors promoted to float64).
    """
    sign = -1.0 if j & 1 else 1.0
    pw = power
    if k == 0:
        val = pw(rho, m) * ch[0]
    elif k == 1:
        s1 = derivative_scale(j, m, 0, 1)
        val = m * pw(rho, max(m - 1, 0)) * ch[0] - 4.0 * s1 * pw(rho, m + 1) * ch[1]
    elif k == 2:
        s1 = derivative_scale(j, m, 0, 1)
        s2 = derivative_scale(j, m, 0, 2)
        val = ((m - 1) * m * pw(rho, max(m - 2, 0)) * ch[0]
               - 4.0 * (2 * m + 1) * s1 * pw(rho, m) * ch[1]
               + 16.0 * s2 * pw(rho, m + 2) * ch[2])
    elif k == 3:
        s1 = derivative_scale(j, m, 0, 1)
        s2 = derivative_scale(j, m, 0, 2)
        s3 = derivative_scale(j, m, 0, 3)
        val = ((m - 2) * (m - 1) * m * pw(rho, max(m - 3, 0)) * ch[0]
               - 12.0 * m * m * s1 * pw(rho, max(m - 1, 0)) * ch[1]
               + 48.0 * (m + 1) * s2 * pw(rho, m + 1) * ch[2]
               - 64.0 * s3 * pw(rho, m + 3) * ch[3])
    else:
        raise ValueError(f"derivative order must be 0..3, got {k}")
    return sign * val


def radial_single(n: int, m_abs: int, rho: np.ndarray, k: int = 0) -> np.ndarray:
    """zk/evaluate.py:157-186: one mode, every shifted chain from degree 0."""
    rho = np.atleast_1d(np.asarray(rho, dtype=np.float64))
    u = jacobi_argument(rho)
    j = (n - m_abs) // 2
    ch = []
    for i in range(k + 1):
        d = j - i
        ch.append(jacobi_chain(d, m_abs + i, i, u)[d] if d >= 0 else np.zeros_like(rho))
    return assemble(rho, m_abs, j, k, ch)


def radial_batch(modes, rho: np.ndarray, k: int = 0, parallel: bool = False,
                 power=numpy_power) -> np.ndarray:
    """zk/batch.py:104-142 (cached strategy) + :97-101 scatter.

    Returns the (P, M) matrix, F-contiguous like the reference's fancy-index
    gather. ``parallel`` maps alpha groups onto a thread pool exactly as the
    reference does (:136-138); results are bitwise independent of it.
    ``power=cr_power`` swaps numpy's pow for the correctly rounded power.
    """
    rho = np.atleast_1d(np.asarray(rho, dtype=np.float64))
    keys, scatter = unique_and_scatter(modes)
    u = jacobi_argument(rho)
    zeros = np.zeros_like(rho)
    unique = np.empty((rho.size, len(keys)), dtype=np.float64)
    groups = groups_by_alpha(keys)

    def run(item):
        a, entries = item
        top = max(j for _, j in entries)
        chains = [jacobi_chain(top - i, a + i, i, u) if top - i >= 0 else None
                  for i in range(k + 1)]
        for slot, j in entries:
            ch = [chains[i][j - i] if j - i >= 0 else zeros for i in range(k + 1)]
            unique[:, slot] = assemble(rho, a, j, k, ch, power)

    if parallel and len(groups) > 1:
        with ThreadPoolExecutor() as pool:
            list(pool.map(run, groups))
    else:
        for g in groups:
            run(g)
    return unique[:, scatter] if scatter else unique


def zernike_2d(n: int, m: int, rho: np.ndarray, theta: np.ndarray, k: int = 0) -> np.ndarray:
    """zk/evaluate.py:259-274: radial x cos(m*theta) (m>=0) / sin(|m|*theta)."""
    rho = np.atleast_1d(np.asarray(rho, dtype=np.float64))
    theta = np.atleast_1d(np.asarray(theta, dtype=np.float64))
    radial = radial_single(n, abs(m), rho, k)
    if m >= 0:
        return radial * np.cos(m * theta)
    return radial * np.sin(abs(m) * theta)


def basis_2d(modes, rho: np.ndarray, theta: np.ndarray, k: int = 0) -> np.ndarray:
    """Column stack of ``zernike_2d`` (the reference's per-mode loop,
    zk/cli.py:438-440), computed through the batch radial matrix so large
    bases stay affordable. Column-wise identical to stacking ``zernike_2d``
    because the batch column equals ``radial_jacobi`` bitwise
    (reference tests/test_batch.py:108-116)."""
    rho = np.atleast_1d(np.asarray(rho, dtype=np.float64))
    theta = np.atleast_1d(np.asarray(theta, dtype=np.float64))
    radial = radial_batch(modes, rho, k)
    out = np.empty_like(radial, order="F")
    for col, (n, m) in enumerate(modes):
        ang = np.cos(m * theta) if m >= 0 else np.sin(abs(m) * theta)
        out[:, col] = radial[:, col] * ang
    return out


# --------------------------------------------------------------------------
# exact oracle (zk/exact.py) -- integer coefficients, one correct rounding
# --------------------------------------------------------------------------

def exact_terms(n: int, m_abs: int, k: int = 0) -> list[tuple[int, int]]:
    """zk/exact.py:48-80: (exponent, integer coefficient), descending, then
    differentiated k times term-wise."""
    from math import comb
    j = (n - m_abs) // 2
    terms = [(n - 2 * s, (-1) ** s * comb(n - s, s) * comb(n - 2 * s, j - s))
             for s in range(j + 1)]
    for _ in range(k):
        terms = [(e - 1, c * e) for e, c in terms if e >= 1]
    return terms


def exact_value(terms, rho: float) -> float:
    """zk/exact.py:92-116: homogenised integer Horner at the exact binary64
    rational rho = a/b, then one correctly rounded division."""
    if not terms:
        return 0.0
    a, b = float(rho).as_integer_ratio()
    top = terms[0][0]
    acc = terms[0][1]
    bpow = 1
    prev = top
    for e, c in terms[1:]:
        gap = prev - e
        bpow *= b ** gap
        acc = acc * a ** gap + c * bpow
        prev = e
    num = acc * a ** prev
    if num == 0:
        return 0.0
    return num / b ** top


def exact_table_rational(modes, points, k: int = 0) -> np.ndarray:
    """exact_table at exact rationals (fractions.Fraction), like the
    reference's accuracy study (zk/cli.py:117-121)."""
    out = np.empty((len(points), len(modes)), dtype=np.float64)
    for col, (n, m) in enumerate(modes):
        t = exact_terms(int(n), abs(int(m)), k)
        for i, p in enumerate(points):
            if not t:
                out[i, col] = 0.0
                continue
            a, b = p.numerator, p.denominator
            top, acc, bpow, prev = t[0][0], t[0][1], 1, t[0][0]
            for e, c in t[1:]:
                bpow *= b ** (prev - e)
                acc = acc * a ** (prev - e) + c * bpow
                prev = e
            num = acc * a ** prev
            out[i, col] = 0.0 if num == 0 else num / b ** top
    return out


def exact_table(modes, rho, k: int = 0) -> np.ndarray:
    """zk/exact.py:129-169: correctly rounded exact values, (P, M)."""
    pts = [float(x) for x in np.atleast_1d(np.asarray(rho, dtype=np.float64))]
    out = np.empty((len(pts), len(modes)), dtype=np.float64)
    cache: dict[tuple[int, int], np.ndarray] = {}
    for col, (n, m) in enumerate(modes):
        key = (int(n), abs(int(m)))
        if key not in cache:
            t = exact_terms(key[0], key[1], k)
            cache[key] = np.array([exact_value(t, x) for x in pts], dtype=np.float64)
        out[:, col] = cache[key]
    return out


@dataclass(frozen=True)
class Workload:
    """Synthetic inputs of BASELINE.json configs."""

    resolution: int
    points: int
    deriv_order: int = 0

    def grid(self) -> np.ndarray:
        # zk/tables.py:46-51 linear_radial_grid
        return np.arange(self.points, dtype=np.float64) / float(self.points - 1)

    def modes(self) -> list[tuple[int, int]]:
        return full_modes(self.resolution)


# --------------------------------------------------------------------------
# binary128 oracle (oracle/zk_quad.c) -- fast high-precision check for big sweeps
# --------------------------------------------------------------------------

_QUAD = None


def _quad_lib():
    """Load (building on first use if needed) oracle/build/libzk_quad.so."""
    global _QUAD
    if _QUAD is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "build", "libzk_quad.so")
        src = os.path.join(here, "zk_quad.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(so), exist_ok=True)
            subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", so,
                            "-lquadmath"], check=True)
        lib = ctypes.CDLL(so)
        p = ctypes.c_void_p
        lib.zkq_radial_table.argtypes = [p, p, ctypes.c_int64, p, ctypes.c_int64, ctypes.c_int, p]
        lib.zkq_radial_table.restype = ctypes.c_int
        _QUAD = lib
    return _QUAD


def quad_table(modes, rho, k: int = 0) -> np.ndarray:
    """(P, M) values computed in binary128 and rounded once (see zk_quad.c)."""
    n = np.ascontiguousarray([int(a) for a, _ in modes], dtype=np.int32)
    m = np.ascontiguousarray([int(b) for _, b in modes], dtype=np.int32)
    r = np.ascontiguousarray(rho, dtype=np.float64)
    out = np.empty((n.size, r.size), dtype=np.float64)
    if n.size and r.size:
        rc = _quad_lib().zkq_radial_table(n.ctypes.data, m.ctypes.data, n.size, r.ctypes.data,
                                          r.size, int(k), out.ctypes.data)
        if rc:
            raise ValueError("bad derivative order")
    return out.T


# --------------------------------------------------------------------------
# float baselines (zk/evaluate.py:189-247), for the GPU baseline kernels
# --------------------------------------------------------------------------

def direct_single(n: int, m_abs: int, rho, k: int = 0) -> np.ndarray:
    """zk/evaluate.py:189-208: Horner in u = rho*rho over coefficients rounded
    once to binary64, times rho**low."""
    rho = np.atleast_1d(np.asarray(rho, dtype=np.float64))
    terms = exact_terms(n, m_abs, k)
    if not terms:
        return np.zeros_like(rho)
    u = rho * rho
    acc = np.full_like(rho, float(terms[0][1]))
    for _, c in terms[1:]:
        acc = acc * u + float(c)
    return acc * rho ** terms[-1][0]


def ztt_table(modes, rho) -> np.ndarray:
    """zk/evaluate.py:211-241: memoised Zernike three-term recursion."""
    rho = np.atleast_1d(np.asarray(rho, dtype=np.float64))
    memo: dict = {}

    def level(n, m):
        if (n, m) in memo:
            return memo[(n, m)]
        v = rho ** n if n == m else rho * (level(n - 1, abs(m - 1)) + level(n - 1, m + 1)) - level(n - 2, m)
        memo[(n, m)] = v
        return v

    out = np.empty((rho.size, len(modes)), dtype=np.float64)
    for c, (n, m) in enumerate(modes):
        out[:, c] = level(int(n), abs(int(m)))
    return out
