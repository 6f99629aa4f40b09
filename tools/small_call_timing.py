"""Per-call wall time of small numpy-level requests (the reference CLI's
`bench` sizes: full mode sets n = 10..100 on 100 / 1000 points), with the
host-side pieces timed separately. Prints one JSON line per (n, P)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402
from paper_2409_19156_b200.evaluate import basis_matrix  # noqa: E402


def med(fn, reps=21):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        fn()
        ts.append(time.perf_counter_ns() - t0)
    return int(np.median(ts))


for P in (100, 1000):
    grid = zb.linear_radial_grid(P)
    for N in range(10, 101, 10):
        modes = zb.full_mode_set(N)
        req = zb.BatchRequest(modes=modes, grid=grid)
        n = np.array([md.n for md in modes], np.int32)
        m = np.array([md.m for md in modes], np.int32)
        ctx = _lib.context(0)
        rec = {"P": P, "N": N, "M": len(modes),
               "evaluate_batch_ns": med(lambda: zb.evaluate_batch(req)),
               "basis_matrix_ns": med(lambda: basis_matrix(n, m, grid, 0)),
               "step_counters_ns": med(lambda: _lib.step_counters(n, m, 0, True)),
               "plan_for_ns": med(lambda: _lib.plan_for(ctx, n, m))}
        print(json.dumps(rec), flush=True)
