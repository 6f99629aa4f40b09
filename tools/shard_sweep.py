"""Per-shard kernel time of config 2 under strong scaling, on ONE GPU: the
shard rank 0 gets when 1e5 points are split over N GPUs (bench.py's
partition), timed exactly as bench.py times a step. This is not a multi-GPU
measurement (no other rank runs); it shows how close each shard stays to the
store roofline as it shrinks -- the ideal aggregate is N x (1e5/N points) x
5151 modes / (the shard's time). Prints one JSON line per N."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

modes = zb.full_mode_set(100)
n, m = zb.modes.mode_arrays(modes)
M = len(modes)
ctx = _lib.context(0)
plan = _lib.plan_for(ctx, n, m)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
grid = zb.linear_radial_grid(100_000)
for world in (1, 2, 4, 8):
    lo, hi = zb.shard_range(100_000, world, 0)
    P = hi - lo
    rho = torch.from_numpy(np.ascontiguousarray(grid[lo:hi])).cuda()
    out = torch.empty((M, P), dtype=torch.float64, device="cuda")
    def step():
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, 0, 0,
                                           out.data_ptr(), P, 0, _lib.ZK_ASYNC), "eval")
    with torch.cuda.stream(stream):
        for _ in range(5):
            step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(reps):
            step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = 8.0 * P * (M + 1) / (ms * 1e-3) / 1e9
    print(json.dumps({"gpus": world, "shard_points": P, "shard_ms": ms, "shard_GBps": gbs,
                      "ideal_aggregate_evals_per_s": 100_000 * M / (ms * 1e-3)}), flush=True)
    del out

# config 5's fit per rank: the series (K3) and the normal equations (K4) on the
# rank's 1e6/N disc points; K5 (one allreduce of 14.3 MB) and K6 (the 1891 x
# 1891 Cholesky) are per-step constants not timed here
modes5 = zb.full_mode_set(60)
n5, m5 = zb.modes.mode_arrays(modes5)
M5 = len(modes5)
plan5 = _lib.plan_for(ctx, n5, m5)
rng = np.random.default_rng(0)
rho5 = np.sqrt(rng.uniform(size=1_000_000))
th5 = 2 * np.pi * rng.uniform(size=1_000_000)
coef5 = torch.from_numpy(rng.standard_normal(M5)).cuda()
for world in (1, 2, 4, 8):
    lo, hi = zb.shard_range(1_000_000, world, 0)
    P = hi - lo
    rho = torch.from_numpy(np.ascontiguousarray(rho5[lo:hi])).cuda()
    th = torch.from_numpy(np.ascontiguousarray(th5[lo:hi])).cuda()
    y = torch.empty(P, dtype=torch.float64, device="cuda")
    G = torch.zeros((M5, M5), dtype=torch.float64, device="cuda")
    r = torch.zeros(M5, dtype=torch.float64, device="cuda")

    def k3():
        _lib.check(_lib.lib.zk_series_eval(ctx.handle, plan5.handle, rho.data_ptr(), th.data_ptr(), P,
                                           0, coef5.data_ptr(), 1, M5, y.data_ptr(), P,
                                           _lib.ZK_ASYNC), "series")

    def k4():
        _lib.check(_lib.lib.zk_gram_accumulate(ctx.handle, plan5.handle, rho.data_ptr(),
                                               th.data_ptr(), P, y.data_ptr(), G.data_ptr(),
                                               r.data_ptr(), _lib.ZK_ASYNC), "gram")

    res = {}
    for name, fn, reps in (("series_ms", k3, 20), ("gram_ms", k4, 3)):
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(reps):
                fn()
        e1.record(stream)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / reps
    print(json.dumps({"c5fit_gpus": world, "shard_points": P, **res,
                      "gram_alg_tflops": P * (M5 + 1) * (M5 + 2) / (res["gram_ms"] * 1e-3) / 1e12}),
          flush=True)
