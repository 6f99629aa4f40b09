"""Hunt for points where the GPU basis differs from the reference algorithm
run with correctly rounded powers (the property test's bitwise claim)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import zk_oracle as orc  # noqa: E402

import paper_2409_19156_b200 as zb  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
special = np.array([0.0, 1.0, 0.5, 1e-300, 5e-324, 2.2250738585072014e-308, 1 - 2 ** -53, 2 ** -30,
                    1e-10, 1e-20, 1e-100, 1e-160, 1e-200, 3e-5, 0.999999, 1e-7,
                    1e-150, 3e-98, 1e-74, 1e-60, 2e-51, 1e-45, 7e-38])
bad_total = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2000):
    nm = int(rng.integers(1, 31))
    modes = []
    for _ in range(nm):
        n = int(rng.integers(0, 61))
        modes.append((n, -n + 2 * int(rng.integers(0, n + 1))))
    npts = int(rng.integers(1, 41))
    pts = rng.uniform(size=npts)
    sel = rng.uniform(size=npts) < 0.4
    pts[sel] = rng.choice(special, size=sel.sum()) * rng.choice([1.0, 1.0, 3.7, 0.77], size=sel.sum())
    pts = np.clip(pts, 0.0, 1.0)
    k = int(rng.integers(0, 4))
    t, _ = zb.evaluate_batch(zb.BatchRequest(modes=zb.as_mode_set(modes), grid=pts, deriv_order=k))
    ref_cr = orc.radial_batch(modes, pts, k, power=orc.cr_power)
    neq = ~((t.values == ref_cr) | (np.isnan(t.values) & np.isnan(ref_cr)))
    if neq.any():
        bad_total += 1
        for p, c in np.argwhere(neq)[:3]:
            print("case", it, "k", k, "mode", modes[c], "rho", repr(pts[p]), "gpu", repr(t.values[p, c]),
                  "ref_cr", repr(ref_cr[p, c]))
print("done; cases with differences:", bad_total)
