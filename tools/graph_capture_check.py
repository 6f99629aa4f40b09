"""Can the device-resident C-ABI calls be captured into a CUDA graph? Captures
one zk_radial_eval (config 2), one zk_zernike_eval and one zk_series_eval on a
torch side stream, replays the graph, and compares with the eager calls
(bitwise) and times replay vs eager launches.
python tools/graph_capture_check.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

modes = zb.full_mode_set(100)
n, m = zb.modes.mode_arrays(modes)
M, P = len(modes), 100_000
ctx = _lib.context(0)
plan = _lib.plan_for(ctx, n, m)
rho = torch.from_numpy(zb.linear_radial_grid(P)).cuda()
th = torch.from_numpy(np.random.default_rng(0).uniform(-3, 3, P)).cuda()
coef = torch.from_numpy(np.random.default_rng(1).standard_normal(M)).cuda()
out = torch.empty(M * P, dtype=torch.float64, device="cuda")
out2 = torch.empty(M * P, dtype=torch.float64, device="cuda")
f = torch.empty(P, dtype=torch.float64, device="cuda")
A = _lib.ZK_ASYNC


def calls():
    _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, 0, 0,
                                       out.data_ptr(), P, 0, A), "radial")
    _lib.check(_lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.data_ptr(), th.data_ptr(), P,
                                        0, 0, out2.data_ptr(), P, 0, A), "2d")
    _lib.check(_lib.lib.zk_series_eval(ctx.handle, plan.handle, rho.data_ptr(), th.data_ptr(), P,
                                       0, coef.data_ptr(), 1, M, f.data_ptr(), P, A), "series")


s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
with torch.cuda.stream(s):
    calls()  # warm-up: plans, scratch, kernel attributes
torch.cuda.synchronize()
eager = (out.clone(), out2.clone(), f.clone())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    calls()
out.zero_(), out2.zero_(), f.zero_()
g.replay()
torch.cuda.synchronize()
same = all(torch.equal(a, b) for a, b in zip(eager, (out, out2, f)))
print("graph replay bitwise equal to eager:", same)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("eager", lambda: calls()), ("graph", lambda: g.replay())):
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        e0.record(s)
        for _ in range(20):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 20:.3f} ms per (radial + 2-D + series)")
