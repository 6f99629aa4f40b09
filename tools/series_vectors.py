"""Config-5 series with V coefficient vectors: the FMA-folding kernel
(ZK_SERIES_DMMA=0) vs the DMMA contraction (ZK_SERIES_DMMA=1), device-resident,
CUDA events. python tools/series_vectors.py [V ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

P = 1_000_000
modes = zb.full_mode_set(60)
M = len(modes)
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
for V in [int(v) for v in sys.argv[1:]] or [1, 8, 32, 64]:
    C = torch.from_numpy(rng.standard_normal((M, V))).cuda()
    res = {}
    for path in ("0", "1"):
        os.environ["ZK_SERIES_DMMA"] = path
        f = zb.series_device(modes, C, rho, th)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f = zb.series_device(modes, C, rho, th)
        e1.record()
        torch.cuda.synchronize()
        res[path] = (e0.elapsed_time(e1) / 5, f.clone())
    d = float((res["0"][1] - res["1"][1]).abs().max())
    print(f"V={V:3d}: FMA folding {res['0'][0]:.2f} ms, DMMA {res['1'][0]:.2f} ms, max |diff| {d:.2e}",
          flush=True)
