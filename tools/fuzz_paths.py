"""Randomised cross-path fuzzing of the C ABI on the GPU: every host/device
input/output combination, ld/order-stride padding, all-orders, 2-D, pinned and
pageable host buffers, duplicated / sign-flipped / sparse mode sets, point
counts across chunk boundaries -- all must equal the plain device call
bitwise, and the plain device call must equal the oracle (reference
algorithm with correctly rounded powers) on a sample of points.
Usage: python tools/fuzz_paths.py [seed] [cases]"""
import ctypes
import os
import sys
import time
from fractions import Fraction

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import zk_oracle as orc  # noqa: E402

import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

def run(seed: int, cases: int, verbose: bool = True) -> int:
    """Number of mismatching (case, path) pairs."""
    rng = np.random.default_rng(seed)
    ctx = _lib.context()
    HI, HO = _lib.ZK_HOST_INPUT, _lib.ZK_HOST_OUTPUT
    t_start = time.time()
    bad = 0
    for it in range(cases):
        kind = rng.integers(0, 7)
        if kind == 6:  # very long chains: k = 3 runs the global-coefficient fallback
            modes = []
            for _ in range(int(rng.integers(1, 4))):
                n = int(rng.integers(1800, 3001))
                modes.append((n, -n + 2 * int(rng.integers(0, n + 1))))
        elif kind == 0:
            modes = [(md.n, md.m) for md in zb.full_mode_set(int(rng.integers(0, 70)))]
        else:
            cnt = int(rng.integers(1, 400))
            nmax = int(rng.integers(0, 120))
            modes = []
            for _ in range(cnt):
                n = int(rng.integers(0, nmax + 1))
                modes.append((n, -n + 2 * int(rng.integers(0, n + 1))))
            if kind in (2, 4):  # duplicates and sign flips
                modes += modes[: cnt // 3] + [(n, -m) for n, m in modes[: cnt // 4]]
        ms = zb.as_mode_set(modes)
        n = np.array([md.n for md in ms], np.int32)
        m = np.array([md.m for md in ms], np.int32)
        plan = _lib.plan_for(ctx, n, m)
        M = len(ms)
        P = int(rng.choice([1, 7, 1023, 1024, 1025, int(rng.integers(1, 60000))]))
        if M * P > 40_000_000:
            P = max(1, 40_000_000 // M)
        k = int(rng.integers(0, 4))
        all_orders = bool(rng.integers(0, 2)) and k > 0
        ang = bool(rng.integers(0, 3) == 0)
        NO = k + 1 if all_orders else 1
        rho = rng.uniform(size=P)
        rho[rng.uniform(size=P) < 0.05] = rng.choice([0.0, 1.0, 0.5], size=None)
        th = 2 * np.pi * rng.uniform(size=P) - np.pi
        d_rho = torch.tensor(rho, device="cuda")
        d_th = torch.tensor(th, device="cuda")

        def call(rp, tp, outp, ld, ostride, flags):
            if ang:
                return _lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rp, tp, P, k, int(all_orders),
                                                outp, ld, ostride, flags)
            return _lib.lib.zk_radial_eval(ctx.handle, plan.handle, rp, P, k, int(all_orders), outp,
                                           ld, ostride, flags)

        ref = torch.empty(NO * M * P, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        _lib.check(call(d_rho.data_ptr(), d_th.data_ptr(), ref.data_ptr(), P, M * P, 0), "ref")
        ref_h = ref.cpu().numpy().reshape(NO, M, P)
        # oracle on a few points (order k, or every order)
        idx = np.unique(rng.integers(0, P, size=min(P, 5)))
        for o in range(NO):
            kk = o if all_orders else k
            if ang:
                want = orc.basis_2d([(md.n, md.m) for md in ms], rho[idx], th[idx], kk)
                got = ref_h[o][:, idx].T
                fin = np.isfinite(want)
                same_special = np.array_equal(got[~fin], want[~fin], equal_nan=True)
                scale = np.maximum(1.0, np.abs(np.where(fin, want, 0.0)).max(axis=0))
                ok = same_special and (np.abs(np.where(fin, got - want, 0.0)) / scale
                                       <= 1e-12).all()
            else:
                want = orc.radial_batch([(md.n, md.m) for md in ms], rho[idx], kk, power=orc.cr_power)
                got = ref_h[o][:, idx].T
                tiny = np.abs(want) < 1e-250
                # bitwise only where the power window rho^(|m|+k) >= 2^-916
                # (DESIGN.md section 3); below, the double-double power is
                # within a few subnormal ulps: parity tolerance
                exact = np.array([[float(Fraction(float(r)) ** (abs(md.m) + k)) >= 2.0 ** -916
                                   for md in ms] for r in rho[idx]])
                # (NaN where the reference algorithm itself overflows: a chain
                # P_j^(a,b) beyond 1e308 times an underflowed rho^m -> 0 * inf)
                sel = ~tiny & exact
                fin = np.isfinite(want)
                err = np.abs(np.where(fin, got - want, 0.0))
                ok = (np.array_equal(got[sel], want[sel], equal_nan=True)
                      and np.array_equal(np.isfinite(got), fin)
                      and (err <= 1e-13 + 1e-12 * np.abs(np.where(fin, want, 0.0))).all())
            if not ok:
                bad += 1
                print("ORACLE MISMATCH", it, M, P, k, all_orders, ang, "| kind", int(kind),
                      "| modes", modes[:3], "| rho", rho[idx][:3])
                if verbose:
                    sel = sel if not ang else np.ones_like(got, bool)
                    diff = sel & ~((got == want) | (np.isnan(got) & np.isnan(want)))
                    for pi, ci in list(zip(*np.nonzero(diff)))[:6]:
                        print(f"   order {kk} point rho={rho[idx][pi]!r} mode {ms[ci].n},{ms[ci].m}: "
                              f"gpu {got[pi, ci]!r} oracle {want[pi, ci]!r}")
        # every other path
        ld = P + int(rng.integers(0, 3))
        ostride = ld * M + int(rng.integers(0, 5))
        total = (NO - 1) * ostride + ld * M
        for flags in (HI, HO, HI | HO):
            host_in = bool(flags & HI)
            rp = rho.ctypes.data if host_in else d_rho.data_ptr()
            tp = th.ctypes.data if host_in else d_th.data_ptr()
            if flags & HO:
                if rng.integers(0, 2):
                    buf = ctypes.c_void_p()
                    _lib.check(_lib.lib.zk_host_alloc(8 * total, ctypes.byref(buf)), "alloc")
                    out = np.ctypeslib.as_array(ctypes.cast(buf.value, ctypes.POINTER(ctypes.c_double)),
                                                shape=(total,))
                else:
                    buf = None
                    out = np.empty(total)
                out[:] = np.nan
                _lib.check(call(rp, tp, out.ctypes.data, ld, ostride, flags), "host out")
                res = out
            else:
                buf = None
                dout = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
                torch.cuda.synchronize()
                _lib.check(call(rp, tp, dout.data_ptr(), ld, ostride, flags), "dev out")
                res = dout.cpu().numpy()
            for o in range(NO):
                blk = res[o * ostride:o * ostride + ld * M].reshape(M, ld)
                if (not np.array_equal(blk[:, :P], ref_h[o], equal_nan=True)
                        or not np.isnan(blk[:, P:]).all()):
                    bad += 1
                    print("PATH MISMATCH", it, flags, M, P, k, all_orders, ang, ld, ostride,
                          "| value diffs", int((blk[:, :P] != ref_h[o]).sum()),
                          "| pad writes", int((~np.isnan(blk[:, P:])).sum()),
                          "| nan in ref", int(np.isnan(ref_h[o]).sum()), "| kind", int(kind),
                          "| modes", modes[:3])
            if buf is not None:
                del out, res
                _lib.lib.zk_host_free(buf)
    print(f"seed {seed}: {cases} cases, {bad} mismatches, {time.time() - t_start:.0f} s")
    return bad


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 0, int(sys.argv[2]) if len(sys.argv) > 2 else 200)
