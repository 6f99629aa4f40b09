"""Config 5 on the GPU box's HOST with the unmodified reference (baseline/_ref):
the 2-D basis as the reference CLI builds it -- one zernike_eval per mode
(zk/cli.py:438-440) -- then the series B @ c, the normal equations B^T B,
B^T y and np.linalg.solve (numpy/OpenBLAS, all host cores). One repetition
(SURVEY.md §8d). Prints one JSON line; the GPU side of the same workload is
bench.py's c5fit phase and bench_configs.py C5.
Usage: python tools/cpu_c5_reference.py [points=1000000] [n=60]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import zernkit as zk  # noqa: E402  (the unmodified reference)

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
modes = zk.full_mode_set(N)
M = len(modes)
rng = np.random.default_rng(0)  # the same draw as bench.py c5fit / bench_configs C5
rho = np.sqrt(rng.uniform(size=P))
theta = 2 * np.pi * rng.uniform(size=P)
c = rng.standard_normal(M)
B = np.empty((P, M), order="F")
t0 = time.perf_counter()
for col, mode in enumerate(modes):
    B[:, col] = zk.zernike_eval(mode, rho, theta)
t_basis = time.perf_counter() - t0
t0 = time.perf_counter()
f = B @ c
t_series = time.perf_counter() - t0
t0 = time.perf_counter()
G = B.T @ B
r = B.T @ f
t_gram = time.perf_counter() - t0
t0 = time.perf_counter()
x = np.linalg.solve(G, r)
t_solve = time.perf_counter() - t0
try:
    from threadpoolctl import threadpool_info
    blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
except Exception:
    blas = None
print(json.dumps({
    "workload": f"config 5 on the host: full mode set n<={N} ({M} modes), {P} disc points "
                "(rho=sqrt(U), theta=2 pi V, seed 0), the unmodified reference",
    "basis_s": t_basis, "basis_evals_per_s": P * M / t_basis,
    "series_s": t_series, "gram_s": t_gram, "solve_s": t_solve,
    "total_s": t_basis + t_series + t_gram + t_solve,
    "fit_max_abs_err_vs_c": float(np.abs(x - c).max()),
    "cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "blas": blas,
    "basis_path": "one zernike_eval per mode (zk/cli.py:438-440), single Python thread",
}))
