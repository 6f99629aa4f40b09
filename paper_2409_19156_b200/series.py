"""Series evaluation and least-squares fitting in the 2-D / radial Zernike
basis (config 5 of BASELINE.json).

The reference has no series or fit API; its 2-D basis is a per-mode loop of
``zernike_eval`` (zk/cli.py:438-440, zk/evaluate.py:259-274) and the closest
contraction is the orthogonality Gram of tests/test_acceptance.py:150-172.
Here:
  * ``series_eval``  f = B c  -- K3, fused: B is never materialised;
  * ``gram``         G = B^T B, r = B^T y -- K4, fp64 DMMA tensor cores;
  * ``fit``          solve G x = r (Cholesky, cuSOLVER through torch) --
                     K6, off the timed path;
  * ``fit_sharded``  points sharded over ranks, partial G/r summed with one
                     NCCL allreduce (K5), then the same solve on every rank.
Numpy inputs/outputs go through the C ABI's host-buffer paths; torch CUDA
tensors stay on the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .evaluate import _check_order
from .modes import as_mode_set, mode_arrays
from .tables import angular_grid, radial_grid

_HOST = _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT


def _modes(modes):
    ms = as_mode_set(modes)
    n, m = mode_arrays(ms)
    return ms, n, m


def _points(rho, theta):
    r = np.ascontiguousarray(radial_grid(rho))
    if theta is None:
        return r, None
    t = np.ascontiguousarray(angular_grid(theta))
    if t.size != r.size:
        raise ValueError(f"point-wise grids must match: {r.size} radial vs {t.size} angular")
    return r, t


def series_eval(modes, coef, rho, theta=None, deriv_order: int = 0, device: int | None = None):
    """f(p) = sum_col coef[col] * Z_col(rho_p, theta_p) (radial basis when theta is
    None). ``coef`` (M,) -> f (P,); ``coef`` (M, V) -> f (P, V)."""
    ms, n, m = _modes(modes)
    k = _check_order(deriv_order)
    r, t = _points(rho, theta)
    c = np.asarray(coef, dtype=np.float64)
    vec = c.ndim == 1
    c2 = np.asfortranarray(c.reshape(len(ms), -1))
    V = c2.shape[1]
    f = np.zeros((r.size, V), dtype=np.float64, order="F")
    if r.size and V:
        ctx = _lib.context(device)
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_series_eval(ctx.handle, plan.handle, _lib.dptr(r),
                                           _lib.dptr(t) if t is not None else None, r.size, k,
                                           _lib.dptr(c2), V, max(len(ms), 1), _lib.dptr(f),
                                           r.size, _HOST), "zk_series_eval")
    return f[:, 0].copy() if vec else f


def gram(modes, rho, theta=None, y=None, device: int | None = None):
    """Normal equations of the least-squares fit: (G = B^T B, r = B^T y or None)."""
    ms, n, m = _modes(modes)
    r, t = _points(rho, theta)
    M = len(ms)
    G = np.zeros((M, M), dtype=np.float64, order="F")
    Bty = np.zeros(M, dtype=np.float64) if y is not None else None
    yy = None
    if y is not None:
        yy = np.ascontiguousarray(y, dtype=np.float64)
        if yy.shape != (r.size,):
            raise ValueError(f"y must have shape ({r.size},), got {yy.shape}")
    if r.size and M:
        ctx = _lib.context(device)
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_gram_accumulate(
            ctx.handle, plan.handle, _lib.dptr(r), _lib.dptr(t) if t is not None else None,
            r.size, _lib.dptr(yy) if yy is not None else None, _lib.dptr(G),
            _lib.dptr(Bty) if Bty is not None else None, _HOST), "zk_gram_accumulate")
    return G, Bty


# --------------------------------------------------------------------------
# device-resident (torch) entry points
# --------------------------------------------------------------------------

def _device_f64(*named):
    """Device entry points take CUDA float64 tensors on one device; anything
    else would be reinterpreted bytes, so it is rejected up front."""
    import torch
    dev = None
    for name, t in named:
        if t is None:
            continue
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
            raise TypeError(f"{name} must be a CUDA float64 tensor, got "
                            f"{type(t).__name__}{'' if not isinstance(t, torch.Tensor) else ' ' + str(t.dtype) + ' on ' + str(t.device)}")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"{name} is on {t.device}, expected {dev}")


def _torch_ctx(tensor, device):
    import torch
    dev = tensor.device.index if device is None else device
    ctx = _lib.context(dev)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    return ctx


def basis_device(plan_modes, rho, deriv_order: int = 0, theta=None, all_orders: bool = False):
    """The basis of ``plan_modes`` at the CUDA float64 tensor ``rho`` (and
    ``theta`` for the 2-D basis), left on the device: a column-major (P, M)
    tensor view -- or, with ``all_orders``, a list of the k+1 orders 0..k
    from one kernel sweep -- computed on torch's current stream, no host
    copy. Values are bitwise those of the numpy entry points. Zero-copy to
    other frameworks through DLPack (``torch.utils.dlpack.to_dlpack``)."""
    import torch
    _device_f64(("rho", rho), ("theta", theta))
    ms, n, m = _modes(plan_modes)
    k = _check_order(deriv_order)
    M, P = len(ms), rho.numel()
    NO = k + 1 if (all_orders and k > 0) else 1
    rho = rho.contiguous()
    theta = theta.contiguous() if theta is not None else None
    out = torch.empty((NO, M, P), dtype=torch.float64, device=rho.device)
    if P and M:
        ctx = _torch_ctx(rho, None)
        plan = _lib.plan_for(ctx, n, m)
        if theta is None:
            rc = _lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, k,
                                         int(NO > 1), out.data_ptr(), P, P * M, _lib.ZK_ASYNC)
        else:
            rc = _lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.data_ptr(),
                                          theta.data_ptr(), P, k, int(NO > 1), out.data_ptr(),
                                          P, P * M, _lib.ZK_ASYNC)
        _lib.check(rc, "zk_radial_eval" if theta is None else "zk_zernike_eval")
    mats = [out[o].t() for o in range(NO)]
    return mats if all_orders else mats[0]


def gram_device(plan_modes, rho, theta=None, y=None, G=None, Bty=None):
    """Accumulate G += B^T B, Bty += B^T y for CUDA tensors (float64) on the
    tensors' device, on torch's current stream. Returns (G, Bty)."""
    import torch
    _device_f64(("rho", rho), ("theta", theta), ("y", y), ("G", G), ("Bty", Bty))
    ms, n, m = _modes(plan_modes)
    M = len(ms)
    dev = rho.device
    if G is None:
        G = torch.zeros((M, M), dtype=torch.float64, device=dev)
    if y is not None and Bty is None:
        Bty = torch.zeros(M, dtype=torch.float64, device=dev)
    rho = rho.contiguous()
    theta = theta.contiguous() if theta is not None else None
    y = y.contiguous() if y is not None else None
    P = rho.numel()
    if P and M:
        ctx = _torch_ctx(rho, None)
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_gram_accumulate(
            ctx.handle, plan.handle, rho.data_ptr(), theta.data_ptr() if theta is not None else None,
            P, y.data_ptr() if y is not None else None, G.data_ptr(),
            Bty.data_ptr() if Bty is not None else None, _lib.ZK_ASYNC), "zk_gram_accumulate")
    return G, Bty


def series_device(plan_modes, coef, rho, theta=None, deriv_order: int = 0):
    """f = B c for CUDA tensors (float64); coef (M,) or (M, V)."""
    import torch
    _device_f64(("rho", rho), ("theta", theta), ("coef", coef))
    ms, n, m = _modes(plan_modes)
    k = _check_order(deriv_order)
    M = len(ms)
    c2 = coef.reshape(M, -1).t().contiguous().t()  # column-major (M, V)
    V = c2.shape[1]
    P = rho.numel()
    f = torch.zeros((V, P), dtype=torch.float64, device=rho.device).t()  # column-major (P, V)
    if P and V:
        ctx = _torch_ctx(rho, None)
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_series_eval(
            ctx.handle, plan.handle, rho.contiguous().data_ptr(),
            theta.contiguous().data_ptr() if theta is not None else None, P, k, c2.data_ptr(), V,
            max(M, 1), f.data_ptr(), P, _lib.ZK_ASYNC), "zk_series_eval")
    return f[:, 0] if coef.dim() == 1 else f


def solve_normal(G, Bty, ridge: float = 0.0):
    """K6: Cholesky solve of (G + ridge I) x = Bty on the GPU (cuSOLVER via
    torch.linalg); off the timed path."""
    import torch
    Gt = torch.as_tensor(G, dtype=torch.float64, device="cuda")
    bt = torch.as_tensor(Bty, dtype=torch.float64, device="cuda")
    if ridge:
        Gt = Gt + ridge * torch.eye(Gt.shape[0], dtype=Gt.dtype, device=Gt.device)
    L = torch.linalg.cholesky(Gt)
    x = torch.cholesky_solve(bt.reshape(-1, 1), L)[:, 0]
    return x


def fit(modes, rho, theta, y, ridge: float = 0.0) -> np.ndarray:
    """Least-squares coefficients of y in the basis (numpy in/out)."""
    G, r = gram(modes, rho, theta, y)
    return solve_normal(G, r, ridge).cpu().numpy()


def allreduce_normal_equations(G, r, group=None):
    """K5: sum the partial normal equations of every rank with ONE collective
    (G and r packed into one buffer): NCCL allreduce over NVLink for CUDA
    tensors, gloo for CPU tensors (tests). G is symmetric, so its memory
    order does not matter. Returns (G, r) summed over the group."""
    import torch
    import torch.distributed as dist
    M = G.shape[0]
    packed = torch.cat([G.reshape(-1), r.reshape(-1)])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    return packed[: M * M].reshape(M, M), packed[M * M:]


def fit_sharded(modes, rho, theta, y, group=None, ridge: float = 0.0):
    """Distributed fit: this rank's point shard (CUDA tensors) -> partial
    G/r on its GPU (K4) -> allreduce (K5) -> identical Cholesky solve on
    every rank (K6). Returns (x, G, r)."""
    G, r = gram_device(modes, rho, theta, y)
    G, r = allreduce_normal_equations(G, r, group)
    return solve_normal(G, r, ridge), G, r
