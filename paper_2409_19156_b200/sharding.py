"""Point sharding across GPUs: radial points are independent,
so rank r of N evaluates one contiguous shard of the grid with no
communication; only the least-squares fit has an exchange step (one
allreduce of the partial normal equations, ``series.allreduce_normal_equations``).
"""

from __future__ import annotations

import os


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of ``total`` points for ``rank`` of
    ``world`` (sizes differ by at most one; every point in exactly one shard)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def dist_env() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 alone)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def radial_basis_shard(modes, rho_global, world: int, rank: int, deriv_order: int = 0,
                       device: int | None = None):
    """This rank's (P_r, M) block of the global basis, as a CUDA tensor
    (column-major) on ``device`` (default: LOCAL_RANK's GPU under torchrun, else
    torch's current device)."""
    import torch

    from . import _lib
    from .modes import as_mode_set, mode_arrays
    from .tables import radial_grid

    ms = as_mode_set(modes)
    n, m = mode_arrays(ms)
    lo, hi = shard_range(len(rho_global), world, rank)
    if device is None:  # this process's GPU: the local rank under torchrun
        device = dist_env()[2] if "LOCAL_RANK" in os.environ else torch.cuda.current_device()
    dev = int(device)
    rho = torch.as_tensor(radial_grid(rho_global[lo:hi]), dtype=torch.float64, device=f"cuda:{dev}")
    P, M = rho.numel(), len(ms)
    out = torch.empty((M, P), dtype=torch.float64, device=rho.device)
    if P and M:
        ctx = _lib.context(dev)
        ctx.use_torch_stream(dev)
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P,
                                           int(deriv_order), 0, out.data_ptr(), P, 0,
                                           _lib.ZK_ASYNC), "zk_radial_eval")
    return out.t(), (lo, hi)
