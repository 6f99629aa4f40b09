"""A/B timing of the config-5 series (one coefficient vector, device-resident,
CUDA events) under environment switches read per call, interleaved rounds.
AB_N / AB_P / AB_V set the mode set n <= N, the point count and the number of
coefficient vectors (default 60, 1e6, 1).
python tools/series_ab.py [VAR=a,b ...]   (default ZK_SERIES_SCALED=0,1)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

P = int(os.environ.get("AB_P", 1_000_000))
modes = zb.full_mode_set(int(os.environ.get("AB_N", 60)))
M = len(modes)
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
NV = int(os.environ.get("AB_V", 1))  # coefficient vectors
c = torch.from_numpy(rng.standard_normal(M) if NV == 1 else
                     np.asfortranarray(rng.standard_normal((M, NV)))).cuda()
specs = sys.argv[1:] or ["ZK_SERIES_SCALED=0,1"]
arms = [("", "")]
for s in specs:
    k, v = s.split("=")
    arms = [(k, x) for x in v.split(",")]
ref = None
res = {a: [] for a in arms}
outs = {}
for rnd in range(5):
    for k, v in arms:
        os.environ[k] = v
        f = zb.series_device(modes, c, rho, th)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f = zb.series_device(modes, c, rho, th)
        e1.record()
        torch.cuda.synchronize()
        res[(k, v)].append(e0.elapsed_time(e1) / 10)
        outs[(k, v)] = f.clone()
base = outs[arms[0]]
for a in arms:
    d = float((outs[a] - base).abs().max() / base.abs().max())
    print(f"{a[0]}={a[1]}: median {np.median(res[a]):.4f} ms  min {min(res[a]):.4f}  "
          f"max|f-f0|/max|f0| {d:.2e}")
