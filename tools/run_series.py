"""Launch the fused series kernel on config 5 a few times (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
modes = zb.full_mode_set(N)
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
c = torch.from_numpy(rng.standard_normal(len(modes))).cuda()
for _ in range(3):
    f = zb.series_device(modes, c, rho, th)
torch.cuda.synchronize()
print("ok", float(f[:4].sum()))
