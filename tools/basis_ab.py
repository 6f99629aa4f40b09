"""A/B timing of one device-resident basis launch (K1 radial or K2 2-D) under
environment switches read per call, interleaved rounds, CUDA events.
AB_N (modes n <= N, default 60), AB_P (points, 1e6), AB_K (order, 0),
AB_2D (1: 2-D disc basis, default; 0: radial linear grid).
python tools/basis_ab.py VAR=a,b"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

N = int(os.environ.get("AB_N", 60))
P = int(os.environ.get("AB_P", 1_000_000))
K = int(os.environ.get("AB_K", 0))
two_d = os.environ.get("AB_2D", "1") != "0"
modes = zb.full_mode_set(N)
n_arr, m_arr = zb.modes.mode_arrays(modes)
M = len(modes)
ctx = _lib.context(0)
plan = _lib.plan_for(ctx, n_arr, m_arr)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)  # launches and events on one stream
rng = np.random.default_rng(0)
if two_d:
    rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
    th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
else:
    rho = torch.from_numpy(zb.linear_radial_grid(P)).cuda()
out = torch.empty(M * P, dtype=torch.float64, device="cuda")


def call():
    if two_d:
        _lib.check(_lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.data_ptr(), th.data_ptr(),
                                            P, K, 0, out.data_ptr(), P, 0, _lib.ZK_ASYNC), "2d")
    else:
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, K, 0,
                                           out.data_ptr(), P, 0, _lib.ZK_ASYNC), "radial")


k, v = sys.argv[1].split("=")
arms = v.split(",")
res = {a: [] for a in arms}
ref = None
for rnd in range(5):
    for a in arms:
        os.environ[k] = a
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        res[a].append(e0.elapsed_time(e1) / 5)
        if rnd == 0:
            if ref is None:
                ref = out.clone()
            else:
                assert torch.equal(out, ref), f"{k}={a} output differs from {k}={arms[0]}"
for a in arms:
    t = float(np.median(res[a]))
    print(f"N={N} P={P} k={K} 2d={int(two_d)} {k}={a}: median {t:.4f} ms "
          f"({8.0 * M * P / t / 1e6:.0f} GB/s written)")
