"""Zernike mode indexing -- the reference's L0 contract, host side.

Mirrors zk/modes.py (names, ordering, exception classes) so callers of the
reference find the same API. Validation stays in Python and happens before
any native call; the dedup plan itself is computed by the native planner
(``zk_plan_describe``), which is the same code that lays out the device plan,
so indexing seen by the user and by the kernels cannot diverge.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib


class ModeError(ValueError):
    """(n, m) does not index a Zernike polynomial (zk/modes.py:14-15)."""


class DegreeViolation(ModeError):
    """n < 0 (zk/modes.py:18-19)."""


class BoundViolation(ModeError):
    """|m| > n (zk/modes.py:22-23)."""


class ParityViolation(ModeError):
    """n - |m| odd (zk/modes.py:26-27)."""


@dataclass(frozen=True)
class Mode:
    """Validated (n, m) pair; invariants of zk/modes.py:37-43."""

    n: int
    m: int

    def __post_init__(self):
        n, m = self.n, self.m
        if n < 0:
            raise DegreeViolation(f"radial degree must be >= 0, got n={n}")
        if abs(m) > n:
            raise BoundViolation(f"|m| must not exceed n, got (n={n}, m={m})")
        if (n - abs(m)) & 1:
            raise ParityViolation(f"n - |m| must be even, got (n={n}, m={m})")

    @property
    def m_abs(self) -> int:
        return abs(self.m)

    @property
    def jacobi_degree(self) -> int:
        return (self.n - abs(self.m)) // 2


ModeSet = tuple[Mode, ...]


def make_mode(n: int, m: int) -> Mode:
    """zk/modes.py:58-64."""
    return Mode(int(n), int(m))


def as_mode_set(pairs: Iterable) -> ModeSet:
    """zk/modes.py:67-76: Mode instances pass through, pairs are validated."""
    return tuple(p if isinstance(p, Mode) else make_mode(*p) for p in pairs)


def full_mode_set(resolution: int) -> ModeSet:
    """zk/modes.py:79-92: n ascending, then m ascending in steps of 2."""
    resolution = int(resolution)
    if resolution < 0:
        raise DegreeViolation(f"resolution must be >= 0, got {resolution}")
    return tuple(Mode(n, m) for n in range(resolution + 1) for m in range(-n, n + 1, 2))


def mode_arrays(modes: Sequence[Mode]) -> tuple[np.ndarray, np.ndarray]:
    """(n, m) int32 column arrays of a ModeSet, the C ABI's mode format."""
    n = np.fromiter((md.n for md in modes), dtype=np.int32, count=len(modes))
    m = np.fromiter((md.m for md in modes), dtype=np.int32, count=len(modes))
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
