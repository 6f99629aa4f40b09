"""Launch the secondary kernels a few times each (for ncu captures):
  dmma     series on DMMA, C5 with 64 coefficient vectors
  chain    jacobi_chain export, 1e6 points x 100 degrees
  direct   radial_direct float baseline, n <= 40 full set x 1e6 points
  ztt      radial_ztt_table float baseline, n <= 40 x 1e6 points
  dd       double-double reference, n <= 100 x 1e4 points
Usage: python tools/run_misc.py WHAT"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

what = sys.argv[1]
rng = np.random.default_rng(0)
for _ in range(3):
    if what == "dmma":
        modes = zb.full_mode_set(60)
        P = 1_000_000
        rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
        th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
        c = torch.from_numpy(rng.standard_normal((len(modes), 64))).cuda()
        zb.series_device(modes, c, rho, th)
    elif what == "chain":
        zb.jacobi_chain(100, 3, 1, rng.uniform(-1, 1, size=1_000_000))
    elif what == "direct":
        modes = zb.full_mode_set(40)
        zb.radial_direct_table(modes, zb.linear_radial_grid(1_000_000))
    elif what == "ztt":
        modes = zb.full_mode_set(40)
        zb.radial_ztt_table(modes, zb.linear_radial_grid(1_000_000))
    elif what == "dd":
        from paper_2409_19156_b200.accuracy import rational_grid_dd, reference_table
        hi, lo = rational_grid_dd(10_000)
        reference_table(zb.full_mode_set(100), hi, lo, 0)
    torch.cuda.synchronize()
print("ok", what)
