"""Radial-basis throughput across problem sizes (device-resident, CUDA events):
points P at n = 100, and degree n at P = 1e5 -- is the kernel at the store
roofline beyond the BASELINE configs? Prints one JSON line per case."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

ctx = _lib.context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)


def case(N, P, k=0, reps=10):
    modes = zb.full_mode_set(N)
    n, m = zb.modes.mode_arrays(modes)
    plan = _lib.plan_for(ctx, n, m)
    M = len(modes)
    rho = torch.from_numpy(zb.linear_radial_grid(P)).cuda()
    out = torch.empty(M * P, dtype=torch.float64, device="cuda")

    def fn():
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, k, 0,
                                           out.data_ptr(), P, P * M, _lib.ZK_ASYNC), "radial")
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    gbs = (8.0 * P * M + 8.0 * P) / t / 1e9
    print(json.dumps({"n": N, "modes": M, "P": P, "k": k, "ms": t * 1e3, "evals_per_s": P * M / t,
                      "GB_s": gbs, "output_GB": 8.0 * P * M / 1e9}), flush=True)
    del out
    torch.cuda.empty_cache()


for P in (10_000, 30_000, 100_000, 300_000, 1_000_000, 3_000_000):
    case(100, P)
for N in (20, 50, 150, 200, 300, 400):
    case(N, 100_000)
