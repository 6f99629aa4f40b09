"""Wall time of the numpy-level API (host arrays in, fresh numpy matrix out)."""
import os
import sys
import time


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
P = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
modes = zb.full_mode_set(N)
grid = zb.linear_radial_grid(P)
req = zb.BatchRequest(modes=modes, grid=grid)
zb.evaluate_batch(req)
for _ in range(3):
    t0 = time.perf_counter()
    t, _ = zb.evaluate_batch(req)
    dt = time.perf_counter() - t0
    print(f"evaluate_batch n={N} P={P}: {dt*1e3:.1f} ms, {t.values.nbytes/dt/1e9:.1f} GB/s, "
          f"{t.values.size/dt:.3e} evals/s")
