"""B200-native Zernike radial basis (fp64 Jacobi recursion) -- drop-in for
the hot path of the reference package ``zernkit``.

The public names below keep the reference's spelling and semantics
(zk/__init__.py:10-100) for everything on the evaluation path; the values
come from hand-written sm_100a CUDA kernels behind the C ABI in
``include/zk_b200.h``. Importing this package requires the in-tree library
(``paper_2409_19156_b200/lib/libzk_b200.so``); there is no CPU fallback.
"""

from . import accuracy
from .baselines import radial_direct, radial_direct_table, radial_ztt, radial_ztt_table
from .batch import (
    STRATEGIES,
    BatchRequest,
    StepCounter,
    batch_cached,
    batch_independent,
    cached_step_counter,
    evaluate_batch,
    evaluate_batch_all_orders,
    independent_step_counter,
)
from .evaluate import (
    MAX_DERIV_ORDER,
    jacobi_argument,
    jacobi_chain,
    jacobi_derivative_scale,
    jacobi_recursion_steps,
    radial_at_zero,
    radial_jacobi,
    zernike_basis,
    zernike_eval,
    zernike_radial,
)
from .modes import (
    BoundViolation,
    DedupPlan,
    DegreeViolation,
    Mode,
    ModeError,
    ModeSet,
    ParityViolation,
    as_mode_set,
    dedup_plan,
    full_mode_set,
    make_mode,
)
from .series import (
    allreduce_normal_equations,
    fit,
    fit_sharded,
    gram,
    basis_device,
    gram_device,
    pack_normal_equations,
    series_device,
    unpack_normal_equations,
    series_eval,
    solve_normal,
)
from .sharding import radial_basis_shard, shard_range
from .tables import (
    EvalMatrix,
    GridError,
    angular_grid,
    linear_radial_grid,
    radial_grid,
    rational_radial_grid,
)

__version__ = "0.1.0"


def release_buffers() -> None:
    """Give back host and device memory the library caches between calls: the
    recycled numpy result buffers (hostpool) and every context's device
    scratch, page-locked staging ring and bounce buffers
    (zk_ctx_release_buffers). Everything is re-allocated on demand."""
    from . import _lib, hostpool
    hostpool.release()
    with _lib._ctx_lock:
        ctxs = list(_lib._contexts.values())
    for ctx in ctxs:
        ctx.release_buffers()

__all__ = [
    "BatchRequest", "BoundViolation", "DedupPlan", "DegreeViolation", "EvalMatrix",
    "GridError", "MAX_DERIV_ORDER", "Mode", "ModeError", "ModeSet", "ParityViolation",
    "STRATEGIES", "StepCounter", "angular_grid", "as_mode_set", "batch_cached",
    "batch_independent", "cached_step_counter", "dedup_plan", "evaluate_batch",
    "evaluate_batch_all_orders", "full_mode_set", "independent_step_counter",
    "jacobi_argument", "jacobi_chain", "jacobi_derivative_scale", "jacobi_recursion_steps",
    "linear_radial_grid", "make_mode", "radial_at_zero", "radial_grid", "radial_jacobi",
    "rational_radial_grid", "zernike_basis", "zernike_eval", "zernike_radial",
    "series_eval", "series_device", "basis_device", "gram", "gram_device", "fit", "fit_sharded",
    "solve_normal", "allreduce_normal_equations", "pack_normal_equations",
    "unpack_normal_equations", "shard_range", "radial_basis_shard",
    "radial_direct", "radial_direct_table", "radial_ztt", "radial_ztt_table",
    "release_buffers",
]
