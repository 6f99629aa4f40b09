"""Time the C5 Gram (K2 panels + DMMA SYRK + reduce) device-resident with CUDA
events: python tools/time_gram.py [P] [reps]; ZK_LIB selects a library build."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
modes = zb.full_mode_set(60)
M = len(modes)
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
y = torch.from_numpy(rng.standard_normal(P)).cuda()
G = torch.zeros((M, M), dtype=torch.float64, device="cuda")
r = torch.zeros(M, dtype=torch.float64, device="cuda")
zb.gram_device(modes, rho, th, y, G, r)
torch.cuda.synchronize()
G0 = G.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    G.zero_()
    r.zero_()
    zb.gram_device(modes, rho, th, y, G, r)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = 1.0 * P * (M + 1) * (M + 2)
print(f"{os.environ.get('ZK_LIB', 'default')}: {ms:.2f} ms, {alg / ms / 1e9:.2f} TFLOP/s alg, "
      f"bitwise-repeat {bool(torch.equal(G, G0))}")
