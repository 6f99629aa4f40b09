"""Launch one radial-basis configuration a few times (for ncu captures).
Usage: python tools/run_config.py N P k [all_orders] [reps] [2d]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

N, P, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
all_orders = len(sys.argv) > 4 and sys.argv[4] == "1"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
two_d = len(sys.argv) > 6 and sys.argv[6] == "1"
modes = zb.full_mode_set(N)
n, m = zb.modes.mode_arrays(modes)
ctx = _lib.context(0)
plan = _lib.plan_for(ctx, n, m)
M = len(modes)
NO = k + 1 if all_orders else 1
rho = torch.from_numpy(np.sqrt(np.random.default_rng(0).uniform(size=P)) if two_d
                       else zb.linear_radial_grid(P)).cuda()
th = torch.from_numpy(2 * np.pi * np.random.default_rng(1).uniform(size=P)).cuda()
out = torch.empty(NO * M * P, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(reps):
    if two_d:
        rc = _lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.data_ptr(), th.data_ptr(), P, k,
                                      int(all_orders), out.data_ptr(), P, P * M, 0)
    else:
        rc = _lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, k, int(all_orders),
                                     out.data_ptr(), P, P * M, 0)
    _lib.check(rc, "eval")
torch.cuda.synchronize()
print("ok", N, P, k, all_orders, two_d)
