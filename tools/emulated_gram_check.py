"""The opt-in fp64-emulated Gram (gram_emulated.py: int8 slices, tcgen05 int8
GEMMs) against the DMMA Gram: error relative to |B|^T|B| (from the DMMA run's
own |B|, computed on the GPU) and device time, at a small size and config 5.
python tools/emulated_gram_check.py [P] [N]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import gram_emulated as ge  # noqa: E402
from paper_2409_19156_b200 import series as zs  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
S = int(os.environ.get("EMUL_S", 8))
modes = zb.full_mode_set(N)
M = len(modes)
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
y = torch.from_numpy(rng.standard_normal(P)).cuda()
G = torch.zeros((M, M), dtype=torch.float64, device="cuda")
r = torch.zeros(M, dtype=torch.float64, device="cuda")
zs.gram_device(modes, rho, th, y, G, r)
torch.cuda.synchronize()
t0 = time.perf_counter()
Ge, re_ = ge.gram_emulated_device(modes, rho, th, y, slices=S)
torch.cuda.synchronize()
print(f"first call (incl. JIT): {time.perf_counter() - t0:.1f} s", flush=True)
# |B|^T |B| scale from the basis itself (device)
B = zb.basis_device(modes, rho, theta=th)  # (P, M)
absB = B.abs()
scale = absB.t() @ absB
rscale = absB.t() @ y.abs()
del B, absB
errG = float(((Ge - G).abs() / scale).max())
errr = float(((re_ - r).abs() / rscale).max())
print(f"P={P} N={N} M={M} S={S}: max |G_emul - G_dmma| / (|B|^T|B|) = {errG:.2e}, "
      f"Bty {errr:.2e}", flush=True)
for name, fn in (("dmma", lambda: zs.gram_device(modes, rho, th, y, G.zero_(), r.zero_())),
                 ("emulated", lambda: ge.gram_emulated_device(modes, rho, th, y, slices=S))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
