"""Generate golden vectors from the REAL reference (``zernkit``).

Run in the build container only (it needs ``/root/reference``):

    python tests/golden/make_golden.py

Writes ``tests/golden/zk_golden.npz``. The GPU box never runs this script;
it only reads the committed fixture. Every array is produced by calling the
reference's public API, unmodified:

* ``c1_*``  full set n<=20 on linear_radial_grid(1000) (config 1), k=0 at all
  points, k=1..3 at every 4th point;
* ``c2_*``  full set n<=100 on a subsample of linear_radial_grid(10**5) plus
  uniform-random points (configs 2/3);
* ``c4_*``  full set n<=200 on a subsample of linear_radial_grid(10**4), with
  the reference's exact oracle on the same points (config 4);
* ``c5_*``  2-D basis n<=60 at disc points (config 5) via per-mode
  ``zernike_eval`` (reference zk/cli.py:438-440 pattern), derivative orders
  0..3, and f = B @ c;
* ``chain_*`` jacobi_chain rows for shifted (alpha, beta), x in [-1, 1];
* ``base_*`` the float baselines radial_direct (k <= 2) and radial_ztt_table;
* ``idx_*`` mode indexing: full_mode_set, dedup plans of mixed requests,
  step counters.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "zk_golden.npz")


def unique_cols(modes):
    """Column indices of the first appearance of each (n,|m|) key."""
    seen, cols = set(), []
    for c, md in enumerate(modes):
        key = (md.n, md.m_abs)
        if key not in seen:
            seen.add(key)
            cols.append(c)
    return np.array(cols, dtype=np.int64)


def batch(zk, modes, grid, k):
    from zernkit.batch import BatchRequest, evaluate_batch
    table, counter = evaluate_batch(BatchRequest(modes=modes, grid=grid, deriv_order=k))
    return table.values, counter


def main():
    sys.path.insert(0, REF)
    import zernkit as zk

    rng = np.random.default_rng(0)
    g = {}

    # ---- config 1
    modes = zk.full_mode_set(20)
    grid = zk.linear_radial_grid(1000)
    ucols = unique_cols(modes)
    g["c1_ucols"] = ucols
    for k in range(4):
        pts = grid if k == 0 else grid[::4]
        vals, counter = batch(zk, modes, pts, k)
        g[f"c1_k{k}"] = vals[:, ucols]
        g[f"c1_k{k}_counter"] = np.array([counter.recursion_steps, counter.chain_count])
    g["c1_grid_k0"] = grid
    g["c1_grid_k123"] = grid[::4]

    # ---- configs 2/3
    modes = zk.full_mode_set(100)
    P = 100_000
    idx = np.unique(np.concatenate([[0, 1, 2, P // 2, P - 2, P - 1],
                                    rng.integers(0, P, size=42)]))
    full = zk.linear_radial_grid(P)
    pts = np.concatenate([full[idx], rng.uniform(0.0, 1.0, size=16)])
    ucols = unique_cols(modes)
    g["c2_ucols"] = ucols
    g["c2_grid"] = pts
    for k in range(4):
        p = pts if k == 0 else pts[::4]
        vals, counter = batch(zk, modes, p, k)
        g[f"c2_k{k}"] = vals[:, ucols]
        g[f"c2_k{k}_counter"] = np.array([counter.recursion_steps, counter.chain_count])

    # ---- config 4 (+ exact oracle on the same points)
    modes = zk.full_mode_set(200)
    P = 10_000
    idx = np.unique(np.concatenate([[0, P - 1], rng.integers(0, P, size=14)]))
    pts = zk.linear_radial_grid(P)[idx]
    ucols = unique_cols(modes)
    umodes = tuple(modes[c] for c in ucols)
    vals, counter = batch(zk, modes, pts, 0)
    g["c4_ucols"] = ucols
    g["c4_grid"] = pts
    g["c4_k0"] = vals[:, ucols]
    g["c4_k0_counter"] = np.array([counter.recursion_steps, counter.chain_count])
    g["c4_exact"] = zk.oracle_table(umodes, pts, 0).values

    # ---- config 5 (2-D basis at disc points, series f = B c)
    modes = zk.full_mode_set(60)
    npts = 48
    rho = np.sqrt(rng.uniform(0.0, 1.0, size=npts))
    theta = 2.0 * np.pi * rng.uniform(0.0, 1.0, size=npts)
    B = np.empty((npts, len(modes)), order="F")
    for c, md in enumerate(modes):
        B[:, c] = zk.zernike_eval(md, rho, theta)
    coef = rng.standard_normal(len(modes))
    g["c5_rho"] = rho
    g["c5_theta"] = theta
    g["c5_B"] = B
    g["c5_coef"] = coef
    g["c5_f"] = B @ coef
    B1 = np.empty((npts, len(modes)), order="F")
    for c, md in enumerate(modes):
        B1[:, c] = zk.zernike_eval(md, rho, theta, 1)
    g["c5_B_k1"] = B1
    for k in (2, 3):  # higher radial-derivative orders of the 2-D basis
        Bk = np.empty((npts, len(modes)), order="F")
        for c, md in enumerate(modes):
            Bk[:, c] = zk.zernike_eval(md, rho, theta, k)
        g[f"c5_B_k{k}"] = Bk

    # ---- mode indexing
    fm = zk.full_mode_set(200)
    g["idx_full200"] = np.array([(md.n, md.m) for md in fm], dtype=np.int32)
    reqs = []
    for r in range(6):
        cnt = int(rng.integers(1, 40))
        ns = [int(n) for n in rng.integers(0, 30, size=cnt)]
        pairs = [(n, -n + 2 * int(rng.integers(0, n + 1))) for n in ns]
        pairs += pairs[: cnt // 3]  # duplicates
        pairs += [(n, -m) for n, m in pairs[: cnt // 4]]  # sign flips
        modes_r = zk.as_mode_set(pairs)
        plan = zk.dedup_plan(modes_r)
        g[f"idx_req{r}"] = np.array([(md.n, md.m) for md in modes_r], dtype=np.int32)
        g[f"idx_req{r}_keys"] = np.array(plan.unique_keys, dtype=np.int32).reshape(-1, 2)
        g[f"idx_req{r}_scatter"] = np.array(plan.scatter, dtype=np.int32)
        from zernkit.batch import cached_step_counter, independent_step_counter
        cs = [(cached_step_counter(plan, k).recursion_steps, cached_step_counter(plan, k).chain_count,
               independent_step_counter(plan, k).recursion_steps,
               independent_step_counter(plan, k).chain_count) for k in range(4)]
        g[f"idx_req{r}_counters"] = np.array(cs, dtype=np.int64)
        grid = zk.linear_radial_grid(33)
        for k in (0, 2):
            vals, _ = batch(zk, modes_r, grid, k)
            g[f"idx_req{r}_k{k}"] = vals
    g["idx_req_grid"] = zk.linear_radial_grid(33)

    # ---- jacobi_chain (zk/evaluate.py:36-76) for shifted parameters
    crng = np.random.default_rng(8)
    cx = np.concatenate([[-1.0, 1.0, 0.0], crng.uniform(-1.0, 1.0, size=21)])
    g["chain_x"] = cx
    chain_cases = [(0, 0, 0), (1, 3, 0), (40, 0, 0), (25, 7, 1), (30, 12, 2), (18, 50, 3)]
    g["chain_cases"] = np.array(chain_cases, dtype=np.int32)
    for jm, al, be in chain_cases:
        g[f"chain_{jm}_{al}_{be}"] = zk.jacobi_chain(jm, al, be, cx)

    # ---- the float baselines (zk/evaluate.py:189-247) at mixed points
    brng = np.random.default_rng(7)
    bpts = np.concatenate([[0.0, 1.0, 0.5], brng.uniform(0.0, 1.0, size=29)])
    bmodes = [(n, m) for n in range(0, 41, 3) for m in range(n % 2, n + 1, 4)]
    g["base_pts"] = bpts
    g["base_modes"] = np.array(bmodes, dtype=np.int32)
    for k in (0, 1, 2):
        g[f"base_direct_k{k}"] = np.stack(
            [zk.radial_direct(n, m, bpts, k) for n, m in bmodes], axis=1)
    g["base_ztt"] = zk.radial_ztt_table(zk.as_mode_set(bmodes), bpts)

    # ---- the reference's accuracy study (zk/cli.py:98-130), all methods, k <= 1
    from zernkit.cli import METHODS, run_accuracy
    rows = run_accuracy(24, METHODS, 100, 1, serial=True)
    g["acc_rows"] = np.array([(r.n, r.m, r.deriv_order, METHODS.index(r.method)) for r in rows],
                             dtype=np.int32)
    g["acc_err"] = np.array([r.max_abs_err for r in rows])

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", len(g), "arrays")


if __name__ == "__main__":
    main()
