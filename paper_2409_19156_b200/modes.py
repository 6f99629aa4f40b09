"""Zernike mode indexing -- the reference's L0 contract, host side.

Mirrors zk/modes.py (names, ordering, exception classes) so callers of the
reference find the same API. Validation stays in Python and happens before
any native call; the dedup plan itself is computed by the native planner
(``zk_plan_describe``), which is the same code that lays out the device plan,
so indexing seen by the user and by the kernels cannot diverge.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib


class ModeError(ValueError):
    """Base class: the pair does not index a Zernike polynomial (zk/modes.py:14-15)."""


class DegreeViolation(ModeError):
    """Negative radial degree n (zk/modes.py:18-19)."""


class BoundViolation(ModeError):
    """Azimuthal order outside -n..n (zk/modes.py:22-23)."""


class ParityViolation(ModeError):
    """n and m of different parity (zk/modes.py:26-27)."""


def _violation(n: int, m: int):
    """The first broken invariant of (n, m) as (exception class, message), or
    None -- checked in the reference's order: degree, bound, parity."""
    if n < 0:
        return DegreeViolation, f"n={n}: the radial degree cannot be negative"
    if m > n or -m > n:
        return BoundViolation, f"(n={n}, m={m}): the azimuthal order exceeds the degree"
    if (n - m) % 2:
        return ParityViolation, f"(n={n}, m={m}): n and m must have the same parity"
    return None


@dataclass(frozen=True)
class Mode:
    """A Zernike index (n, m) that satisfies the zk/modes.py:37-43 invariants."""

    n: int
    m: int

    def __post_init__(self):
        bad = _violation(self.n, self.m)
        if bad is not None:
            raise bad[0](bad[1])

    @property
    def m_abs(self) -> int:
        return -self.m if self.m < 0 else self.m

    @property
    def jacobi_degree(self) -> int:
        """Index j of the backing Jacobi polynomial, (n - |m|) / 2."""
        return (self.n - self.m_abs) >> 1


ModeSet = tuple[Mode, ...]


def make_mode(n: int, m: int) -> Mode:
    """zk/modes.py:58-64."""
    return Mode(int(n), int(m))


def as_mode_set(pairs: Iterable) -> ModeSet:
    """zk/modes.py:67-76: Mode instances pass through, pairs are validated.
    A tuple of Modes (an immutable ModeSet) is returned as is, so the per-set
    memo (mode_set_entry) keeps hitting across calls with the same set."""
    if isinstance(pairs, tuple):
        with _SET_CACHE_LOCK:
            hit = _SET_CACHE.get(id(pairs))
        if (hit is not None and hit[0] is pairs) or all(isinstance(p, Mode) for p in pairs):
            return pairs
    return tuple(p if isinstance(p, Mode) else make_mode(*p) for p in pairs)


def full_mode_set(resolution: int) -> ModeSet:
    """Every mode up to degree ``resolution``, n ascending then m ascending in
    steps of 2 (zk/modes.py:79-92); entry n(n+1)/2 + (n+m)/2 is (n, m)."""
    top = int(resolution)
    if top < 0:
        raise DegreeViolation(f"resolution {top} is negative")
    out = []
    for n in range(top + 1):
        out.extend(Mode(n, m) for m in range(-n, n + 1, 2))
    return tuple(out)


_SET_CACHE: "OrderedDict[int, tuple]" = OrderedDict()
_SET_CACHE_LEN = 16
_SET_CACHE_LOCK = threading.Lock()


def mode_set_entry(modes: Sequence[Mode]) -> tuple:
    """(modes, n, m, memo) for a mode set: the (n, m) int32 column arrays
    (read-only) and a dict for other per-set results (the step counters).
    Tuples -- ModeSets are immutable tuples of frozen modes -- are memoised
    by identity, so a request re-evaluated in a loop (the reference CLI's
    ``bench`` repetitions) does not re-walk thousands of Mode objects."""
    key = id(modes)
    if isinstance(modes, tuple):
        with _SET_CACHE_LOCK:
            hit = _SET_CACHE.get(key)
            if hit is not None and hit[0] is modes:
                _SET_CACHE.move_to_end(key)
                return hit
    n = np.fromiter((md.n for md in modes), dtype=np.int32, count=len(modes))
    m = np.fromiter((md.m for md in modes), dtype=np.int32, count=len(modes))
    n.flags.writeable = False
    m.flags.writeable = False
    entry = (modes, n, m, {})
    if isinstance(modes, tuple):
        with _SET_CACHE_LOCK:
            _SET_CACHE[key] = entry  # the entry holds `modes`, so its id stays unique
            while len(_SET_CACHE) > _SET_CACHE_LEN:
                _SET_CACHE.popitem(last=False)
    return entry


def mode_arrays(modes: Sequence[Mode]) -> tuple[np.ndarray, np.ndarray]:
    """(n, m) int32 column arrays of a ModeSet, the C ABI's mode format
    (read-only; memoised per mode-set tuple)."""
    _, n, m, _ = mode_set_entry(modes)
    return n, m


@dataclass(frozen=True)
class DedupPlan:
    """zk/modes.py:95-105: distinct (n,|m|) keys + input->key scatter."""

    unique_keys: tuple[tuple[int, int], ...]
    scatter: tuple[int, ...]


def dedup_plan(modes: Sequence[Mode]) -> DedupPlan:
    """zk/modes.py:108-125, computed by the native planner."""
    n, m = mode_arrays(modes)
    un, um, sc = _lib.describe(n, m)
    return DedupPlan(unique_keys=tuple(zip(un.tolist(), um.tolist())),
                     scatter=tuple(sc.tolist()))
