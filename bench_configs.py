"""Per-config measurements of every BASELINE.json config on one B200.

bench.py is the driver contract (config 2, one JSON line). This script
times each config's hot path device-resident (inputs in HBM, CUDA events on
the launching stream, warm-up first) and reports it against the binding
roofline, so DESIGN.md / profiles/ can cite every config:

  C1  n=20  x 1e3 points, k=0        (launch-bound; parity config)
  C2  n=100 x 1e5 points, k=0
  C3  n=100 x 1e5 points, k=1,2,3 one order per launch, and orders 0..3 in one sweep
  C4  n=200 x 1e4 points, k=0
  C5  2-D n=60 x 1e6 disc points: basis (15.1 GB), fused series f = B c,
      Gram B^T B + B^T y (DMMA), Cholesky solve

Peaks: HBM copy from MEASURED_PEAKS.json (6549.8 GB/s this round), HBM write-only 7321 GB/s
(cudaMemset, tools/hbm_write_probe.cu), FP64 36.9 TFLOP/s (DMMA/DFMA,
tools/fp64_peak_probe.cu).

Usage: python bench_configs.py [--only C2,C5] [--out profiles/r01_configs.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _copy_peak(default=6549.8):
    """HBM copy GB/s from the driver-written MEASURED_PEAKS.json (rewritten each round)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return default


HBM_COPY = _copy_peak()
HBM_WRITE = 7321.0
FP64 = 36.9e12


def main():
    import torch

    import paper_2409_19156_b200 as zb
    from paper_2409_19156_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    only = set(args.only.split(","))
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_copy = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm_copy = HBM_COPY

    ctx = _lib.context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    results = []

    def timed(fn, reps, warm=3):
        with torch.cuda.stream(stream):
            for _ in range(warm):
                fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    def plan_of(modes):
        n, m = zb.modes.mode_arrays(modes)
        return _lib.plan_for(ctx, n, m), n, m

    def counters(modes, k):
        n, m = zb.modes.mode_arrays(modes)
        steps, chains = _lib.step_counters(n, m, k, True)
        un, um, _ = _lib.describe(n, m)
        return steps, chains, un.size

    def alg_flops(P, modes, k, orders):
        steps, chains, U = counters(modes, k)
        A = {0: 3, 1: 8, 2: 12, 3: 16}
        return P * (3 + 6 * steps + 4 * chains + sum(A[o] for o in orders) * U)

    def radial_case(name, N, P, k, all_orders=False, reps=args.reps):
        modes = zb.full_mode_set(N)
        plan, n, m = plan_of(modes)
        M = len(modes)
        NO = k + 1 if all_orders else 1
        rho = torch.from_numpy(zb.linear_radial_grid(P)).cuda()
        out = torch.empty(NO * M * P, dtype=torch.float64, device="cuda")

        def fn():
            _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, k,
                                               int(all_orders), out.data_ptr(), P, P * M,
                                               _lib.ZK_ASYNC), "radial")

        t = timed(fn, reps)
        nbytes = 8.0 * P * M * NO + 8.0 * P
        orders = list(range(k + 1)) if all_orders else [k]
        fl = alg_flops(P, modes, k, orders)
        rec = {"config": name, "N": N, "P": P, "M": M, "deriv_order": k, "orders_written": NO,
               "ms": t * 1e3, "evals_per_s": P * M * NO / t,
               "hbm_gbs": nbytes / t / 1e9, "frac_hbm_copy_peak": nbytes / t / 1e9 / hbm_copy,
               "frac_hbm_write_peak": nbytes / t / 1e9 / HBM_WRITE,
               "alg_fp64_tflops": fl / t / 1e12, "frac_fp64": fl / t / FP64,
               "bound": "hbm" if nbytes / (hbm_copy * 1e9) > fl / FP64 else "fp64"}
        del out
        torch.cuda.empty_cache()
        return rec

    if "C1" in only:
        results.append(radial_case("C1", 20, 1000, 0, reps=200))
    if "C2" in only:
        results.append(radial_case("C2", 100, 100_000, 0))
    if "C3" in only:
        for k in (1, 2, 3):
            results.append(radial_case(f"C3 k={k}", 100, 100_000, k))
        results.append(radial_case("C3 orders 0..3", 100, 100_000, 3, all_orders=True, reps=10))
    if "C4" in only:
        results.append(radial_case("C4", 200, 10_000, 0))
    if "C5" in only:
        modes = zb.full_mode_set(60)
        plan, n, m = plan_of(modes)
        M = len(modes)
        P = 1_000_000
        rng = np.random.default_rng(0)
        rho_h = np.sqrt(rng.uniform(size=P))
        th_h = 2 * np.pi * rng.uniform(size=P)
        coef_h = rng.standard_normal(M)
        rho = torch.from_numpy(rho_h).cuda()
        th = torch.from_numpy(th_h).cuda()
        coef = torch.from_numpy(coef_h).cuda()
        out = torch.empty(M * P, dtype=torch.float64, device="cuda")

        def basis():
            _lib.check(_lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.data_ptr(),
                                                th.data_ptr(), P, 0, 0, out.data_ptr(), P, 0,
                                                _lib.ZK_ASYNC), "zernike")

        t = timed(basis, 5)
        nbytes = 8.0 * P * M + 16.0 * P
        results.append({"config": "C5 2-D basis", "N": 60, "P": P, "M": M, "ms": t * 1e3,
                        "evals_per_s": P * M / t, "hbm_gbs": nbytes / t / 1e9,
                        "frac_hbm_copy_peak": nbytes / t / 1e9 / hbm_copy,
                        "frac_hbm_write_peak": nbytes / t / 1e9 / HBM_WRITE, "bound": "hbm"})
        del out
        torch.cuda.empty_cache()
        f = torch.empty(P, dtype=torch.float64, device="cuda")

        def series():
            _lib.check(_lib.lib.zk_series_eval(ctx.handle, plan.handle, rho.data_ptr(),
                                               th.data_ptr(), P, 0, coef.data_ptr(), 1, M,
                                               f.data_ptr(), P, _lib.ZK_ASYNC), "series")

        t = timed(series, 10)
        steps, chains, U = counters(modes, 0)
        fl = P * (3 + 6 * steps + 4 * chains + 3 * U + 3 * M)  # + angular mul and fma per column
        results.append({"config": "C5 series f=Bc (fused)", "P": P, "M": M, "ms": t * 1e3,
                        "evals_per_s": P * M / t, "alg_fp64_tflops": fl / t / 1e12,
                        "frac_fp64": fl / t / FP64, "bound": "fp64",
                        "note": "B never materialised; materialise+GEMV would move 2x15.1 GB. "
                                "alg_fp64 is the SURVEY 8d count (6 FP64 ops per exact "
                                "recursion step); the scaled recursion executes 2 per step, so "
                                "it can exceed the FP64 peak -- the FP64 pipe utilisation is "
                                "in the ncu capture (profiles/r02/kernels.md)"})
        y = torch.empty(P, dtype=torch.float64, device="cuda")
        series()
        torch.cuda.synchronize()
        y.copy_(f)
        G = torch.zeros((M, M), dtype=torch.float64, device="cuda")
        r = torch.zeros(M, dtype=torch.float64, device="cuda")

        def gram():
            G.zero_()
            r.zero_()
            _lib.check(_lib.lib.zk_gram_accumulate(ctx.handle, plan.handle, rho.data_ptr(),
                                                   th.data_ptr(), P, y.data_ptr(), G.data_ptr(),
                                                   r.data_ptr(), _lib.ZK_ASYNC), "gram")

        t = timed(gram, 3, warm=1)
        bm = 64  # G block edge of the SYRK tiles (zk_gram.cu BM; 128 in round 1)
        nb = (M + 1 + bm - 1) // bm
        exe = 2.0 * P * (nb * (nb + 1) // 2) * bm * bm
        alg = 1.0 * P * (M + 1) * (M + 2)  # triangle of [B y]^T [B y]
        results.append({"config": "C5 Gram B^T B + B^T y (DMMA)", "P": P, "M": M, "ms": t * 1e3,
                        "alg_fp64_tflops_triangle": alg / t / 1e12,
                        "executed_fp64_tflops": exe / t / 1e12, "frac_fp64": exe / t / FP64,
                        "bound": "fp64 (DMMA)", "full_gram_equiv_tflops": 2.0 * P * M * M / t / 1e12})
        zb.solve_normal(G, r)  # warm-up: cuSOLVER handle creation
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = zb.solve_normal(G, r)
        torch.cuda.synchronize()
        ts = time.perf_counter() - t0
        err = float((x - coef).abs().max())
        results.append({"config": "C5 Cholesky solve (cuSOLVER via torch)", "M": M,
                        "ms": ts * 1e3, "max_abs_coef_error": err})

    for r in results:
        print(json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
