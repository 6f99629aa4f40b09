"""Bitwise A/B of two builds of the library on seeded random requests.
Usage: python tools/stress_compare.py OUT.npz            (current ZK_LIB)
       python tools/stress_compare.py --cmp A.npz B.npz  (report differences)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cases(seed=0, count=400):
    rng = np.random.default_rng(seed)
    for c in range(count):
        nm = int(rng.integers(1, 30))
        modes = []
        for _ in range(nm):
            n = int(rng.integers(0, 61))
            modes.append((n, -n + 2 * int(rng.integers(0, n + 1))))
        npts = int(rng.integers(1, 3000))
        pts = rng.uniform(size=npts)
        if c % 3 == 0:
            pts[: npts // 4] = rng.choice([0.0, 1.0, 0.5, 1e-300, 1 - 2 ** -53], size=npts // 4)
        yield modes, pts, int(rng.integers(0, 4))


def main():
    if sys.argv[1] == "--cmp":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        bad = 0
        for key in a.files:
            x, y = a[key], b[key]
            if not np.array_equal(x, y):
                bad += 1
                d = np.argwhere(x != y)
                print(key, "differs at", len(d), "entries; first", d[:3].tolist(),
                      x[tuple(d[0])], y[tuple(d[0])])
        print("cases", len(a.files), "differing", bad)
        return
    import paper_2409_19156_b200 as zb
    out = {}
    for i, (modes, pts, k) in enumerate(cases()):
        t, _ = zb.evaluate_batch(zb.BatchRequest(modes=zb.as_mode_set(modes), grid=pts,
                                                 deriv_order=k))
        out[f"c{i}_k{k}"] = t.values
    np.savez(sys.argv[1], **out)


if __name__ == "__main__":
    main()
