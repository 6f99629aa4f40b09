"""Drop-in installer: route an imported ``zernkit`` package's hot path
through the B200 kernels.

The reference has no operator registry or FFI; its boundary for this path is
five module attributes: ``radial_jacobi`` (zk/evaluate.py:157),
``zernike_eval`` (zk/evaluate.py:259), ``batch_cached`` (zk/batch.py:104),
``batch_independent`` (zk/batch.py:145) and ``evaluate_batch``
(zk/batch.py:184), re-exported by zk/__init__.py:10-36 and bound by
zk/cli.py:21,23. ``install(zernkit)`` rebinds every one of those names to a
wrapper that validates with the reference's own types (its BatchRequest,
Mode, GridError...), computes on the GPU, and returns the reference's own
result types (its EvalMatrix and StepCounter), so callers cannot tell the
difference except for speed. ``uninstall`` restores the originals.

Usage (e.g. from a pytest plugin loaded with ``-p`` before test modules bind
the names):

    import zernkit
    from paper_2409_19156_b200.zernkit_plugin import install
    install(zernkit)
"""

from __future__ import annotations

import importlib

import numpy as np

_SAVED: dict = {}

_TARGETS = {
    "evaluate": ("radial_jacobi", "zernike_eval"),
    "batch": ("batch_cached", "batch_independent", "evaluate_batch"),
    "cli": ("evaluate_batch", "zernike_eval"),
    "": ("radial_jacobi", "zernike_eval", "batch_cached", "batch_independent", "evaluate_batch"),
}


def _wrappers(zk):
    from . import _lib
    from .evaluate import basis_matrix, parallel_devices
    from .modes import mode_set_entry

    ref_eval = importlib.import_module(zk.__name__ + ".evaluate")
    ref_batch = importlib.import_module(zk.__name__ + ".batch")
    ref_tables = importlib.import_module(zk.__name__ + ".tables")
    ref_modes = importlib.import_module(zk.__name__ + ".modes")
    orig = {name: getattr(ref_eval, name) for name in _TARGETS["evaluate"]}
    orig.update({name: getattr(ref_batch, name) for name in _TARGETS["batch"]})


    def radial_jacobi(n, m_abs, grid, deriv_order=0):
        # validation exactly as zk/evaluate.py:173-176, with the reference's types
        if m_abs < 0:
            raise ValueError("m_abs must be non-negative")
        mode = ref_modes.make_mode(n, m_abs)
        if deriv_order not in (0, 1, 2, 3):
            raise ValueError(f"derivative order must be 0..3, got {deriv_order}")
        rho = ref_tables.radial_grid(grid)
        col = basis_matrix(np.array([mode.n], np.int32), np.array([mode.m_abs], np.int32),
                           rho, int(deriv_order))
        return col[:, 0]  # the (P, 1) result is one contiguous column: no copy

    def zernike_eval(mode, grid, angles, deriv_order=0):
        rho = ref_tables.radial_grid(grid)
        theta = ref_tables.angular_grid(angles)
        if rho.size != theta.size:
            raise ValueError(
                f"point-wise grids must match: {rho.size} radial vs {theta.size} angular")
        ref_modes.make_mode(mode.n, mode.m_abs)
        if deriv_order not in (0, 1, 2, 3):
            raise ValueError(f"derivative order must be 0..3, got {deriv_order}")
        col = basis_matrix(np.array([mode.n], np.int32), np.array([mode.m], np.int32), rho,
                           int(deriv_order), theta=theta)
        return col[:, 0]  # the (P, 1) result is one contiguous column: no copy

    def _run(request, shared, parallel):
        # parallel=True: the reference's thread pool (zk/batch.py:136-141)
        # becomes point shards over every visible GPU; bitwise the same values
        # mode arrays and counters memoised per mode-set tuple (modes.py)
        _, n, m, memo = mode_set_entry(request.modes)
        values = basis_matrix(n, m, request.grid, request.deriv_order,
                              devices=parallel_devices() if parallel else None)
        key = ("ref_counter", int(request.deriv_order), bool(shared))
        counter = memo.get(key)
        if counter is None:
            steps, chains = _lib.step_counters(n, m, request.deriv_order, shared)
            counter = memo[key] = ref_batch.StepCounter(recursion_steps=steps,
                                                        chain_count=chains)
        table = ref_tables.EvalMatrix(values=values, modes=request.modes,
                                      deriv_order=request.deriv_order)
        return table, counter

    def batch_cached(request, parallel=False):
        if request.strategy != "cached":
            raise ValueError(f"request strategy is {request.strategy!r}, expected 'cached'")
        return _run(request, True, parallel)

    def batch_independent(request, parallel=False):
        if request.strategy != "independent":
            raise ValueError(
                f"request strategy is {request.strategy!r}, expected 'independent'")
        return _run(request, False, parallel)

    def evaluate_batch(request, parallel=False):
        if request.strategy == "cached":
            return batch_cached(request, parallel)
        return batch_independent(request, parallel)

    new = {"radial_jacobi": radial_jacobi, "zernike_eval": zernike_eval,
           "batch_cached": batch_cached, "batch_independent": batch_independent,
           "evaluate_batch": evaluate_batch}
    return new, orig


def install(zk) -> dict:
    """Rebind the hot-path names of the imported ``zernkit`` package ``zk``.
    Returns the mapping {module.attr: replacement}."""
    new, orig = _wrappers(zk)
    done = {}
    for sub, names in _TARGETS.items():
        modname = zk.__name__ + ("." + sub if sub else "")
        try:
            mod = importlib.import_module(modname)
        except ImportError:  # e.g. the CLI needs click
            continue
        for name in names:
            if hasattr(mod, name):
                _SAVED.setdefault((modname, name), getattr(mod, name))
                setattr(mod, name, new[name])
                done[f"{modname}.{name}"] = new[name]
    return done


def uninstall(zk) -> None:
    """Restore every attribute ``install`` replaced."""
    for (modname, name), fn in list(_SAVED.items()):
        if modname == zk.__name__ or modname.startswith(zk.__name__ + "."):
            setattr(importlib.import_module(modname), name, fn)
            del _SAVED[(modname, name)]
