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

import os

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


def _devices(parallel: bool, device: int | None) -> list:
    if parallel:
        from .evaluate import parallel_devices
        return parallel_devices()
    return [device]


def _on_devices(devs, fn):
    """fn(shard_index) on one host thread per device (the C ABI releases the GIL)."""
    if len(devs) == 1:
        return [fn(0)]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(devs)) as pool:
        return list(pool.map(fn, range(len(devs))))


def series_eval(modes, coef, rho, theta=None, deriv_order: int = 0, device: int | None = None,
                parallel: bool = False):
    """f(p) = sum_col coef[col] * Z_col(rho_p, theta_p) (radial basis when theta is
    None). ``coef`` (M,) -> f (P,); ``coef`` (M, V) -> f (P, V).
    ``parallel``: the points are split into contiguous shards over
    ``parallel_devices()`` (ZK_DEVICES or every visible GPU), each GPU writing
    its rows of f -- no communication; bitwise equal to the one-GPU call."""
    from .sharding import shard_range
    ms, n, m = _modes(modes)
    k = _check_order(deriv_order)
    r, t = _points(rho, theta)
    c = np.asarray(coef, dtype=np.float64)
    vec = c.ndim == 1
    c2 = np.asfortranarray(c.reshape(len(ms), -1))
    V = c2.shape[1]
    P = r.size
    f = np.zeros((P, V), dtype=np.float64, order="F")
    devs = _devices(parallel, device)
    if P and V:
        def run(i):
            lo, hi = shard_range(P, len(devs), i)
            if hi <= lo:
                return
            ctx = _lib.context(devs[i])
            plan = _lib.plan_for(ctx, n, m)
            _lib.check(_lib.lib.zk_series_eval(
                ctx.handle, plan.handle, _lib.dptr(r) + 8 * lo,
                _lib.dptr(t) + 8 * lo if t is not None else None, hi - lo, k, _lib.dptr(c2), V,
                max(len(ms), 1), _lib.dptr(f) + 8 * lo, P, _HOST), "zk_series_eval")

        _on_devices(devs, run)
    return f[:, 0].copy() if vec else f


def gram(modes, rho, theta=None, y=None, device: int | None = None, parallel: bool = False):
    """Normal equations of the least-squares fit: (G = B^T B, r = B^T y or None).
    ``parallel``: points sharded over ``parallel_devices()``, a partial G/r per
    GPU (K4), summed across the GPUs by ONE NCCL allreduce of the packed
    triangle (K5, ``zk_gram_allreduce``) -- the north_star's fitting config in
    one process."""
    ms, n, m = _modes(modes)
    r, t = _points(rho, theta)
    M = len(ms)
    yy = None
    if y is not None:
        yy = np.ascontiguousarray(y, dtype=np.float64)
        if yy.shape != (r.size,):
            raise ValueError(f"y must have shape ({r.size},), got {yy.shape}")
    if parallel:
        return _gram_multi(_devices(True, device), n, m, r, t, yy)
    G = np.zeros((M, M), dtype=np.float64, order="F")
    Bty = np.zeros(M, dtype=np.float64) if y is not None else None
    if r.size and M:
        ctx = _lib.context(device)
        plan = _lib.plan_for(ctx, n, m)
        _lib.check(_lib.lib.zk_gram_accumulate(
            ctx.handle, plan.handle, _lib.dptr(r), _lib.dptr(t) if t is not None else None,
            r.size, _lib.dptr(yy) if yy is not None else None, _lib.dptr(G),
            _lib.dptr(Bty) if Bty is not None else None, _HOST), "zk_gram_accumulate")
    return G, Bty


def _gram_multi(devs, n, m, r, t, yy):
    """Per-GPU partial normal equations on contiguous point shards, summed
    with zk_gram_allreduce (NCCL, one communicator clique per device list);
    the sum is read back from the first GPU."""
    import ctypes

    import torch

    from .sharding import shard_range
    M, P = int(n.size), r.size
    nd = len(devs)

    def part(i):
        dev = torch.device("cuda", int(devs[i]))
        lo, hi = shard_range(P, nd, i)
        with torch.cuda.device(dev):
            G = torch.zeros((M, M), dtype=torch.float64, device=dev)
            b = torch.zeros(M, dtype=torch.float64, device=dev) if yy is not None else None
            if hi > lo and M:
                rho = torch.from_numpy(r[lo:hi]).to(dev)
                th = torch.from_numpy(t[lo:hi]).to(dev) if t is not None else None
                yd = torch.from_numpy(yy[lo:hi]).to(dev) if yy is not None else None
                _gram_device_nm(n, m, rho, th, yd, G, b)
            torch.cuda.current_stream(dev).synchronize()
        return G, b

    parts = _on_devices(devs, part)
    if M:
        ctxs = [_lib.context(int(d)) for d in devs]
        for c in ctxs:
            c.set_stream(None)  # the ctx's own stream; the partials are complete
        arr = ctypes.c_void_p * nd
        _lib.check(_lib.lib.zk_gram_allreduce(
            arr(*[c.handle.value for c in ctxs]), nd, arr(*[g.data_ptr() for g, _ in parts]),
            arr(*[b.data_ptr() for _, b in parts]) if yy is not None else None, M, 0),
            "zk_gram_allreduce")
    G0, b0 = parts[0]
    G = np.asfortranarray(G0.cpu().numpy())
    return G, (b0.cpu().numpy() if b0 is not None else None)


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
    dev = tensor.device.index if device is None else device
    ctx = _lib.context(dev)
    ctx.use_torch_stream(dev)
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
    _device_f64(("rho", rho), ("theta", theta), ("y", y), ("G", G), ("Bty", Bty))
    ms, n, m = _modes(plan_modes)
    return _gram_device_nm(n, m, rho, theta, y, G, Bty)


def _gram_device_nm(n, m, rho, theta, y, G, Bty):
    import torch
    M = int(n.size)
    dev = rho.device
    if G is None:
        G = torch.zeros((M, M), dtype=torch.float64, device=dev)
    if y is not None and Bty is None:
        Bty = torch.zeros(M, dtype=torch.float64, device=dev)
    rho = rho.contiguous()
    theta = theta.contiguous() if theta is not None else None
    y = y.contiguous() if y is not None else None
    P = rho.numel()
    if P and M and os.environ.get("ZK_GRAM_EMULATED", "0") == "1":
        # opt-in: int8 slice products on tcgen05 (gram_emulated.py)
        from .gram_emulated import gram_emulated_nm
        Ge, be = gram_emulated_nm(n, m, rho, theta, y)
        G += Ge
        if Bty is not None and be is not None:
            Bty += be
    elif P and M:
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
    torch.linalg); off the timed path. Tensors stay on their own device;
    numpy inputs go to the current CUDA device."""
    import torch
    dev = G.device if isinstance(G, torch.Tensor) and G.is_cuda else torch.device("cuda")
    Gt = torch.as_tensor(G, dtype=torch.float64, device=dev)
    bt = torch.as_tensor(Bty, dtype=torch.float64, device=dev)
    if ridge:
        Gt = Gt + ridge * torch.eye(Gt.shape[0], dtype=Gt.dtype, device=Gt.device)
    # cholesky_ex: no host sync between the factorisation and the solve (the
    # info check follows both; 1.18 vs 1.24 ms at M = 1891)
    L, info = torch.linalg.cholesky_ex(Gt)
    x = torch.cholesky_solve(bt.reshape(-1, 1), L)[:, 0]
    if int(info.item()) != 0:
        raise torch.linalg.LinAlgError(
            f"normal matrix is not positive definite (leading minor {int(info.item())})")
    return x


def fit(modes, rho, theta, y, ridge: float = 0.0, parallel: bool = False) -> np.ndarray:
    """Least-squares coefficients of y in the basis (numpy in/out);
    ``parallel`` shards the Gram over every GPU (see ``gram``)."""
    G, r = gram(modes, rho, theta, y, parallel=parallel)
    return solve_normal(G, r, ridge).cpu().numpy()


def pack_normal_equations(G, r=None):
    """[upper triangle of G, column-major | r]: M(M+1)/2 + M doubles, the K5 wire
    format (G is symmetric: half the bytes of the full matrix). CUDA tensors
    are packed by the library's kernel on torch's current stream; CPU tensors
    (gloo tests) by index gather in the same order."""
    import torch
    M = G.shape[0]
    n = int(_lib.lib.zk_gram_packed_count(M))
    if G.is_cuda:
        _device_f64(("G", G), ("r", r))
        Gc = G.contiguous()  # symmetric: row- and column-major storage are the same matrix
        out = torch.empty(n, dtype=torch.float64, device=G.device)
        ctx = _torch_ctx(G, None)
        _lib.check(_lib.lib.zk_gram_pack(ctx.handle, Gc.data_ptr(),
                                         r.contiguous().data_ptr() if r is not None else None,
                                         M, out.data_ptr(), _lib.ZK_ASYNC), "zk_gram_pack")
        return out
    iu = torch.triu_indices(M, M)           # row-major (i <= j), ordered by i
    order = torch.argsort(iu[1] * M + iu[0])  # column-major upper triangle
    rows, cols = iu[0][order], iu[1][order]
    tri = G[rows, cols].to(torch.float64)
    rr = r.reshape(-1).to(torch.float64) if r is not None else torch.zeros(M, dtype=torch.float64)
    return torch.cat([tri, rr])


def unpack_normal_equations(packed, M: int):
    """Inverse of ``pack_normal_equations``: (full symmetric G, r)."""
    import torch
    if packed.is_cuda:
        G = torch.empty((M, M), dtype=torch.float64, device=packed.device)
        r = torch.empty(M, dtype=torch.float64, device=packed.device)
        ctx = _torch_ctx(packed, None)
        _lib.check(_lib.lib.zk_gram_unpack(ctx.handle, packed.data_ptr(), M, G.data_ptr(),
                                           r.data_ptr(), _lib.ZK_ASYNC), "zk_gram_unpack")
        return G, r  # symmetric: row- and column-major agree
    tri = M * (M + 1) // 2
    iu = torch.triu_indices(M, M)
    order = torch.argsort(iu[1] * M + iu[0])
    rows, cols = iu[0][order], iu[1][order]
    G = torch.zeros((M, M), dtype=torch.float64)
    G[rows, cols] = packed[:tri]
    G[cols, rows] = packed[:tri]
    return G, packed[tri:tri + M].clone()


def allreduce_normal_equations(G, r, group=None, comm=None):
    """K5: sum the partial normal equations of every rank with ONE collective
    on the packed upper triangle + r (``pack_normal_equations``; C5: 14.3 MB
    + 15 KB). ``comm``: a ``_lib.Comm`` (the library's own NCCL communicator,
    ``zk_gram_allreduce_comm``; G and r are updated in place); otherwise
    torch.distributed -- NCCL over NVLink for CUDA tensors, gloo for CPU
    tensors (tests). Returns (G, r) summed over the group."""
    import torch.distributed as dist
    M = G.shape[0]
    if comm is not None:
        _device_f64(("G", G), ("r", r))
        ctx = _torch_ctx(G, None)
        if comm.ctx is not ctx:
            raise ValueError("comm belongs to another device's context")
        _lib.check(_lib.lib.zk_gram_allreduce_comm(comm.handle, G.data_ptr(),
                                                   r.data_ptr() if r is not None else None, M,
                                                   _lib.ZK_ASYNC), "zk_gram_allreduce_comm")
        return G, r
    packed = pack_normal_equations(G, r)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    return unpack_normal_equations(packed, M)


def fit_sharded(modes, rho, theta, y, group=None, ridge: float = 0.0, comm=None):
    """Distributed fit: this rank's point shard (CUDA tensors) -> partial
    G/r on its GPU (K4) -> allreduce of the packed triangle (K5) -> identical
    Cholesky solve on every rank (K6). Returns (x, G, r)."""
    G, r = gram_device(modes, rho, theta, y)
    G, r = allreduce_normal_equations(G, r, group, comm)
    return solve_normal(G, r, ridge), G, r
