"""Opt-in fp64-emulated normal equations on the tcgen05 tensor cores.

The DMMA Gram (K4, ``zk_gram_accumulate``) runs at the FP64 tensor-core
roofline; ``tcgen05.mma`` has no f64 kind. This path trades that roofline for
the int8 one: the fp64 panel [B y] is split into S int8 slices per column
(``zk_emul_colexp`` / ``zk_emul_slices``: column scale 2^e_j, 7 bits per
slice), the slice products A_s^T A_t -- exact int32 sums over at most 524,287
points -- run as int8 -> int32 GEMMs on tcgen05, and ``zk_emul_accumulate``
recombines them in fp64, G_ij = sum_{s+t<=S-1} 2^(e_i+e_j-12-7(s+t)) C_st[i][j]
(DESIGN.md §9). The int8 GEMM is a LIBRARY kernel: the CUTLASS CuTe-DSL
Blackwell persistent dense GEMM shipped in this image, JIT-compiled once per
process (tens of seconds) -- hence opt-in, never the default.

``gram_emulated_device(modes, rho, theta, y)`` -> (G, Bty) like ``gram_device``.
"""
from __future__ import annotations

import importlib.util
import os

from . import _lib
from .series import _modes

_EX = ("flashinfer/data/cutlass/examples/python/CuTeDSL/blackwell/dense_gemm_persistent.py")
_GEMM = {}  # (Mp,) -> (module, compiled_fn)
KMAX = 524_160  # points per exact int32 chunk (|a_s a_t| <= 4096: < 2^31 / 4096 = 524,288)


def _example_module():
    import site
    for base in site.getsitepackages():
        path = os.path.join(base, _EX)
        if os.path.exists(path):
            spec = importlib.util.spec_from_file_location("zk_dense_gemm_persistent", path)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    raise RuntimeError("the CuTe-DSL Blackwell dense GEMM (flashinfer's CUTLASS examples) is "
                       "not installed: the emulated Gram is unavailable")


def _cute(t, leading_dim):
    from cutlass.cute.runtime import from_dlpack
    return from_dlpack(t, assumed_align=16).mark_layout_dynamic(leading_dim=leading_dim)


def _gemm(a, b, c, stream_ptr):
    """C (L, Mp, Mp) int32 = A (L, Mp, K) int8 @ B (L, K, Mp) int8 (both K-major),
    batched over L."""
    import cuda.bindings.driver as cuda
    import cutlass
    import cutlass.utils as utils
    a_, b_, c_ = _cute(a, 2), _cute(b, 1), _cute(c, 2)
    tile = os.environ.get("ZK_EMUL_TILE", "256x256")  # 3.0 POPS at C5 (256x128: 2.4-2.7)
    key = (a.shape[1], tile)
    if key not in _GEMM:
        mod = _example_module()
        tm, tn = (int(v) for v in tile.split("x"))
        two = tm == 256  # 256-row tiles are the 2-CTA (cluster 2 x 1) MMA
        cl = (2, 1) if two else (1, 1)
        clusters = utils.HardwareInfo().get_max_active_clusters(cl[0] * cl[1])
        fn = mod.compile_bmm((a.shape[1], b.shape[2], a.shape[2], a.shape[0]), a_, b_, c_,
                             cutlass.Int32, "k", "k", "n", (tm, tn), cl, clusters, two, False,
                             epilogue_op=lambda x: x)
        _GEMM[key] = fn
    _GEMM[key](a_, b_, c_, cuda.CUstream(stream_ptr))


def gram_emulated_device(plan_modes, rho, theta, y, slices: int | None = None):
    """G = B^T B and B^T y of the 2-D basis (theta) or the radial one (theta
    None) on CUDA tensors, through int8 slice products on tcgen05."""
    ms, n, m = _modes(plan_modes)
    return gram_emulated_nm(n, m, rho, theta, y, slices)


def gram_emulated_nm(n, m, rho, theta, y, slices: int | None = None):
    """gram_emulated_device on the C ABI's (n, m) column arrays; y may be None
    (then Bty is None). ``slices`` (default ZK_EMUL_SLICES or 8): 7 bits each;
    the error grows with a column's max-to-typical magnitude ratio (per-column
    scaling). Measured at config 5 against the DMMA Gram, relative to |B|^T|B|:
    S = 8 1.8e-15 (73 ms), S = 7 4.2e-15 (59 ms), S = 6 9.3e-12 (45 ms)."""
    import torch
    if slices is None:
        slices = int(os.environ.get("ZK_EMUL_SLICES", "8"))
    M, P = int(n.size), rho.numel()
    dev = rho.device
    S = int(slices)
    Mp = (M + 1 + 255) // 256 * 256  # whole 256-row tiles of the 2-CTA GEMM (partial ones miscompute)
    nch = max(1, -(-P // KMAX))
    Kc = (-(-P // nch) + 127) // 128 * 128
    Pp = nch * Kc
    ctx = _lib.context(dev.index if dev.index is not None else 0)
    stream = torch.cuda.current_stream(dev)
    ctx.use_torch_stream()  # the legacy default stream too (handle 0 = the ctx's own stream)
    plan = _lib.plan_for(ctx, n, m)
    # row j = column j of [B y]; never read past row M or point P (no zero fill)
    panel = torch.empty((M + 1, Pp), dtype=torch.float64, device=dev)
    rp = rho.contiguous()
    if theta is not None:
        _lib.check(_lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rp.data_ptr(),
                                            theta.contiguous().data_ptr(), P, 0, 0,
                                            panel.data_ptr(), Pp, 0, _lib.ZK_ASYNC), "basis")
    else:
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rp.data_ptr(), P, 0, 0,
                                           panel.data_ptr(), Pp, 0, _lib.ZK_ASYNC), "basis")
    if y is not None:
        panel[M, :P] = y
    else:
        panel[M, :P] = 0.0
    e = torch.zeros(Mp, dtype=torch.int32, device=dev)
    sp = stream.cuda_stream or _lib.CUDA_STREAM_LEGACY
    _lib.check(_lib.lib.zk_emul_colexp(panel.data_ptr(), Pp, P, M + 1, e.data_ptr(), sp), "colexp")
    # chunk-major: every (chunk, slice) a dense Mp x Kc operand (strided row
    # views measured 1.5 vs 2.5 POPS)
    sl = torch.empty((nch, S, Mp, Kc), dtype=torch.int8, device=dev)
    _lib.check(_lib.lib.zk_emul_slices(panel.data_ptr(), Pp, P, M + 1, e.data_ptr(), S,
                                       sl.data_ptr(), Kc, nch, Mp, sp), "slices")
    del panel
    G = torch.zeros((Mp, Mp), dtype=torch.float64, device=dev)  # column-major, ld Mp
    # the slice pairs (s, s + d) with 2s + d <= S - 1, s = 0 .. L_d - 1, are ONE
    # batched GEMM per offset d and point chunk: operands sl[0:L_d] and
    # sl[d:d+L_d] share the batch stride (8 launches per chunk for S = 8)
    L0 = (S - 1) // 2 + 1
    C = torch.empty((L0, Mp, Mp), dtype=torch.int32, device=dev)
    for c in range(nch):
        for d in range(S):
            L = (S - 1 - d) // 2 + 1
            a = sl[c, 0:L]
            b = sl[c, d:d + L].permute(0, 2, 1)
            _gemm(a, b, C[:L], sp)
            for s in range(L):
                _lib.check(_lib.lib.zk_emul_accumulate(
                    C[s].data_ptr(), Mp, M + 1, e.data_ptr(), 12 + 7 * (2 * s + d), int(d > 0),
                    G.data_ptr(), Mp, sp), "accumulate")
    Gc = G.t()  # G was written column-major into a row-major tensor
    return Gc[:M, :M].contiguous(), (Gc[:M, M].contiguous() if y is not None else None)


__all__ = ["gram_emulated_device", "gram_emulated_nm"]
