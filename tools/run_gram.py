"""Run the DMMA Gram on config 5 (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 262_144
modes = zb.full_mode_set(60)
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
y = torch.from_numpy(rng.standard_normal(P)).cuda()
G, r = zb.gram_device(modes, rho, th, y)
torch.cuda.synchronize()
print("ok", float(G[0, 0]))
