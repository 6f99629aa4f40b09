"""The reference CLI's 2-D pattern (zk/cli.py:438-440): one zernike_eval call
per mode over the whole grid, here through the GPU path -- per-call overhead
(plan lookup/creation, host copies) dominates small requests."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
rng = np.random.default_rng(0)
rho = np.sqrt(rng.uniform(size=P))
theta = 2 * np.pi * rng.uniform(size=P)
modes = zb.full_mode_set(N)
zb.zernike_eval(modes[0], rho, theta)
t0 = time.perf_counter()
B = np.empty((P, len(modes)), order="F")
for c, md in enumerate(modes):
    B[:, c] = zb.zernike_eval(md, rho, theta)
dt = time.perf_counter() - t0
t1 = time.perf_counter()
Bb = zb.zernike_basis(rho, theta, np.array([m.n for m in modes]), np.array([m.m for m in modes]))
dt2 = time.perf_counter() - t1
print(f"per-mode loop n<={N} ({len(modes)} modes) x {P} points: {dt:.2f} s "
      f"({1e3 * dt / len(modes):.2f} ms/call); one batched call: {dt2 * 1e3:.0f} ms; "
      f"equal: {np.array_equal(B, Bb)}")
