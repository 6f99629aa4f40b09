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
