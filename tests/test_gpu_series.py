"""GPU parity of K3 (fused series f = B c), K4 (DMMA Gram B^T B, B^T y) and
the fit (K6) against the oracle / golden vectors. Calls go through the C ABI."""

import numpy as np
import pytest

import zk_oracle as orc

pytestmark = pytest.mark.gpu

zb = pytest.importorskip("paper_2409_19156_b200")
torch = pytest.importorskip("torch")


def disc(P, seed):
    rng = np.random.default_rng(seed)
    return np.sqrt(rng.uniform(size=P)), 2 * np.pi * rng.uniform(size=P)


def test_series_matches_golden_config5(golden):
    modes = zb.full_mode_set(60)
    f = zb.series_eval(modes, golden["c5_coef"], golden["c5_rho"], golden["c5_theta"])
    scale = np.abs(golden["c5_B"]) @ np.abs(golden["c5_coef"])
    assert (np.abs(f - golden["c5_f"]) <= 1e-13 * scale + 1e-13).all()


@pytest.mark.parametrize("V", [1, 3, 8, 11])
def test_series_multi_vector_2d(V):
    modes = zb.full_mode_set(25)
    rho, theta = disc(777, V)
    C = np.random.default_rng(V).standard_normal((len(modes), V))
    f = zb.series_eval(modes, C, rho, theta)
    B = orc.basis_2d([(md.n, md.m) for md in modes], rho, theta)
    ref = B @ C
    assert f.shape == (777, V)
    assert np.abs(f - ref).max() <= 1e-12 * np.abs(B).sum(axis=1).max() * np.abs(C).max()


@pytest.mark.parametrize("k", [0, 2, 3])
def test_series_radial_derivatives(k):
    modes = zb.full_mode_set(30)
    rho = zb.linear_radial_grid(500)
    c = np.random.default_rng(k).standard_normal(len(modes))
    f = zb.series_eval(modes, c, rho, None, k)
    B = orc.radial_batch([(md.n, md.m) for md in modes], rho, k)
    scale = np.abs(B) @ np.abs(c)
    assert (np.abs(f - B @ c) <= 1e-12 * scale + 1e-13).all()


def test_gram_matches_numpy_and_is_symmetric():
    modes = zb.full_mode_set(20)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(5000, 1)
    y = np.random.default_rng(2).standard_normal(5000)
    G, r = zb.gram(modes, rho, theta, y)
    B = orc.basis_2d(pairs, rho, theta)
    Gr, rr = B.T @ B, B.T @ y
    assert np.array_equal(G, G.T)
    assert np.abs(G - Gr).max() <= 1e-12 * np.abs(Gr).max()
    assert np.abs(r - rr).max() <= 1e-12 * np.abs(B).sum(axis=0).max() * np.abs(y).max()
    G2, _ = zb.gram(modes, rho, theta, None)
    assert np.array_equal(G2, G)  # y column does not perturb B^T B
    G3, r3 = zb.gram(modes, rho, theta, y)
    assert np.array_equal(G3, G) and np.array_equal(r3, r)  # deterministic


def test_gram_multi_panel_and_partial_tail(monkeypatch):
    modes = zb.full_mode_set(15)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(10_000, 3)
    y = np.random.default_rng(4).standard_normal(10_000)
    B = orc.basis_2d(pairs, rho, theta)
    monkeypatch.setenv("ZK_GRAM_PANEL_MB", "3")  # 3 MB / (256 cols * 8 B) -> 1024-point panels
    G, r = zb.gram(modes, rho, theta, y)
    assert np.abs(G - B.T @ B).max() <= 1e-12 * np.abs(B.T @ B).max()
    assert np.abs(r - B.T @ y).max() <= 1e-11 * np.abs(B.T @ y).max()


def test_gram_radial_basis_and_config5_shape():
    modes = zb.full_mode_set(60)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(20_000, 5)
    G, _ = zb.gram(modes, rho, theta)
    B = orc.basis_2d(pairs, rho, theta)
    Gr = B.T @ B
    assert G.shape == (1891, 1891)
    assert np.abs(G - Gr).max() <= 1e-12 * np.abs(Gr).max()
    Gr2, _ = zb.gram(modes, rho, None)
    Br = orc.radial_batch(pairs, rho, 0)
    assert np.abs(Gr2 - Br.T @ Br).max() <= 1e-12 * np.abs(Br.T @ Br).max()


def test_fit_recovers_coefficients():
    modes = zb.full_mode_set(12)
    rho, theta = disc(20_000, 6)
    c = np.random.default_rng(7).standard_normal(len(modes))
    y = zb.series_eval(modes, c, rho, theta)
    x = zb.fit(modes, rho, theta, y)
    assert np.abs(x - c).max() < 1e-9


def test_device_accumulate_equals_single_call():
    modes = zb.full_mode_set(10)
    rho, theta = disc(4096, 8)
    y = np.random.default_rng(9).standard_normal(4096)
    t = lambda a: torch.tensor(a, dtype=torch.float64, device="cuda")
    G, r = zb.gram_device(modes, t(rho[:2000]), t(theta[:2000]), t(y[:2000]))
    G, r = zb.gram_device(modes, t(rho[2000:]), t(theta[2000:]), t(y[2000:]), G, r)
    Gh, rh = zb.gram(modes, rho, theta, y)
    assert np.abs(G.cpu().numpy() - Gh).max() <= 1e-12 * np.abs(Gh).max()
    assert np.abs(r.cpu().numpy() - rh).max() <= 1e-11 * np.abs(rh).max()
    x, Gs, rs = zb.fit_sharded(modes, t(rho), t(theta), t(y))  # world of one
    assert np.abs(x.cpu().numpy() - np.linalg.solve(Gh, rh)).max() < 1e-8
    f = zb.series_device(modes, x, t(rho), t(theta))
    assert f.shape == (4096,)


@pytest.mark.parametrize("path", ["0", "1"])
@pytest.mark.parametrize("k", [0, 2])
@pytest.mark.parametrize("V", [1, 5, 8, 13])
def test_series_fma_and_dmma_paths(monkeypatch, path, k, V):
    """Both series engines (per-key FMA folding, and the DMMA contraction
    used for several coefficient vectors) against B @ C, 2-D and radial."""
    monkeypatch.setenv("ZK_SERIES_DMMA", path)
    modes = zb.full_mode_set(23)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(1000, V + 7 * k)
    C = np.random.default_rng(V).standard_normal((len(modes), V))
    for th in (theta, None):
        f = zb.series_eval(modes, C, rho, th, k)
        B = orc.basis_2d(pairs, rho, theta, k) if th is not None else orc.radial_batch(pairs, rho, k)
        ref = B @ C
        scale = np.abs(B) @ np.abs(C)
        assert (np.abs(f - ref) <= 1e-13 * scale + 1e-13).all(), (path, k, V, th is None)


ENGINES = {  # single-vector k = 0 series engines (environment switches read per call)
    "resident3": {},
    "resident2": {"ZK_SERIES_K0": "2"},
    "resident4": {"ZK_SERIES_K0": "4"},
    "staged_scaled": {"ZK_SERIES_K0": "0"},
    "staged_unscaled": {"ZK_SERIES_K0": "0", "ZK_SERIES_SCALED": "0"},
    "exact": {"ZK_SERIES_EXACT": "1"},
    "staged_resident": {"ZK_SERIES_K0": "0", "ZK_SERIES_RESIDENT": "1"},
    "staged_vec2": {"ZK_SERIES_K0": "0", "ZK_SERIES_VEC3": "0"},
}


@pytest.mark.parametrize("V", [2, 3, 5, 6, 7])
def test_series_resident_multi_vector_passes(monkeypatch, V):
    """Several vectors on the resident kernel (passes of 2 and 1 vectors, up to
    6) and on the staged kernel (7+): every column against B @ C, 2-D and
    radial, with a point count that is not a tile multiple."""
    modes = zb.full_mode_set(17)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(1237, V)
    C = np.random.default_rng(V).standard_normal((len(modes), V))
    for engine in ("3", "0"):
        monkeypatch.setenv("ZK_SERIES_K0", engine)
        for th in (theta, None):
            f = zb.series_eval(modes, C, rho, th)
            B = orc.basis_2d(pairs, rho, theta) if th is not None else orc.radial_batch(pairs, rho, 0)
            scale = np.abs(B) @ np.abs(C)
            assert f.shape == (1237, V)
            assert (np.abs(f - B @ C) <= 1e-13 * scale + 1e-300).all(), (V, engine, th is None)


@pytest.mark.parametrize("engine", sorted(ENGINES))
def test_series_k0_engines_edge_cases(monkeypatch, engine):
    """Every single-vector k = 0 engine against B @ c of the oracle: the
    resident kernel (zk_series_k0.cu) at 2/3/4 points per thread, the staged
    kernel on scaled and unscaled chains, and the exact arithmetic. Sparse
    alpha sets (rotation steps > 1 and anchors after jumps > 4), a group split
    into virtual groups (> 4096 duplicated columns), rho = 0 and 1, point
    counts that are not tile multiples, 2-D and radial."""
    for k, v in ENGINES[engine].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(5)
    sparse = [(n, m) for n, m in [(0, 0), (1, 1), (7, -1), (9, 3), (12, -2), (30, 8), (31, -9),
                                  (31, 13), (40, 22), (44, -24), (45, 25), (60, 60), (61, -59)]]
    dup = [(6, 2)] * 4200 + [(6, -2)] * 300 + [(5, 1), (9, -3)]
    for pairs in (sparse, dup):
        modes = zb.as_mode_set(pairs)
        c = rng.standard_normal(len(modes))
        for P in (1, 255, 769, 2049):
            rho, theta = disc(P, P)
            rho[0] = 0.0
            if P > 1:
                rho[1] = 1.0
            for th in (theta, None):
                f = zb.series_eval(modes, c, rho, th)
                B = orc.basis_2d(pairs, rho, theta) if th is not None else orc.radial_batch(pairs, rho, 0)
                scale = np.abs(B) @ np.abs(c)
                assert (np.abs(f - B @ c) <= 1e-13 * scale + 1e-300).all(), (engine, len(pairs), P, th is None)
    modes = zb.full_mode_set(8)
    assert zb.series_eval(modes, np.ones(len(modes)), np.zeros(0), np.zeros(0)).shape == (0,)


def test_series_resident_table_too_large_falls_back(monkeypatch):
    """n = 200 (20,301 modes): the key-record table (10,402 rows x 32 B) does not
    fit one CTA's shared memory; the staged kernel takes the request."""
    modes = zb.full_mode_set(200)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(300, 9)
    c = np.random.default_rng(9).standard_normal(len(modes))
    f = zb.series_eval(modes, c, rho, theta)
    B = orc.basis_2d(pairs, rho, theta)
    scale = np.abs(B) @ np.abs(c)
    assert (np.abs(f - B @ c) <= 1e-12 * scale).all()


@pytest.mark.parametrize("V", [1, 3])
def test_series_long_chains_any_degree(V):
    """Chains whose tables exceed the shared-memory stage (n = 3000, k = 3)
    run the global-table variant (the reference has no degree limit,
    zk/evaluate.py:259-274); the stage of several vectors steps down first."""
    modes = zb.as_mode_set([(3000, 0), (2999, -1), (2998, 2), (1200, 0), (7, 3)])
    pairs = [(md.n, md.m) for md in modes]
    rho = np.array([0.0, 0.1, 0.37, 0.5, 0.71, 0.93])
    C = np.random.default_rng(V).standard_normal((len(modes), V))
    for k in (0, 3):
        f = zb.series_eval(modes, C, rho, None, k)
        B = orc.radial_batch(pairs, rho, k)
        scale = np.abs(B) @ np.abs(C)
        assert (np.abs(f.reshape(rho.size, V) - B @ C) <= 1e-12 * scale + 1e-13).all(), k


@pytest.mark.parametrize("N", [60, 100])
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_series_tolerance_mode_error_vs_binary128(monkeypatch, N, k):
    """The series' default tolerance-mode recursion (prescaled coefficients,
    FMA contraction) against the binary128 oracle (oracle/zk_quad.c, bitwise
    the reference's exact oracle on every golden value), next to the exact
    K1-identical arithmetic (ZK_SERIES_EXACT=1): error per point relative to
    sum_col |B c| (2-D basis, fl(|m| theta) angles as zk/evaluate.py:272-274)."""
    modes = zb.full_mode_set(N)
    pairs = [(md.n, md.m) for md in modes]
    rho, theta = disc(1500, N + k)
    c = np.random.default_rng(k).standard_normal(len(modes))
    Bq = orc.quad_table(pairs, rho, k)
    m = np.array([md.m for md in modes])
    ang = np.where(m >= 0, np.cos(np.abs(m)[None, :] * theta[:, None]),
                   np.sin(np.abs(m)[None, :] * theta[:, None]))
    B2 = Bq * ang
    ref = (B2.astype(np.longdouble) @ c.astype(np.longdouble)).astype(np.float64)
    scale = np.abs(B2) @ np.abs(c)
    errs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ZK_SERIES_EXACT", mode)
        f = zb.series_eval(modes, c, rho, theta, k)
        errs[mode] = float((np.abs(f - ref) / scale).max())
    print(f"n<={N} k={k}: tolerance mode {errs['0']:.3e}, exact mode {errs['1']:.3e} "
          f"(of sum|B||c|)")
    assert errs["0"] <= 1e-13
    assert errs["0"] <= 8 * errs["1"] + 1e-15


def test_device_entry_points_reject_wrong_dtype_or_device():
    import torch
    modes = zb.full_mode_set(4)
    rho32 = torch.rand(10, device="cuda", dtype=torch.float32)
    with pytest.raises(TypeError):
        zb.basis_device(modes, rho32)
    with pytest.raises(TypeError):
        zb.series_device(modes, torch.ones(len(modes), dtype=torch.float64), torch.rand(10, dtype=torch.float64))
    with pytest.raises(TypeError):
        zb.gram_device(modes, rho32.double().cpu())


def test_gram_tma_and_cpasync_operand_paths_bitwise(tmp_path):
    """K4's two operand paths -- TMA tensor copies into swizzled tiles through
    an mbarrier ring (default) and the cp.async ring (ZK_GRAM_TMA=0) -- give
    the same bits: same tiles, same DMMA order. 150k points = three panels
    (double-buffered, partials accumulated over panels). The switch is read
    once per process, hence the subprocesses (tools/gram_save.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = tmp_path / f"g{flag}.npy"
        env = dict(os.environ, ZK_GRAM_TMA=flag)
        subprocess.run([sys.executable, os.path.join(root, "tools", "gram_save.py"), str(out),
                        "150000"], check=True, env=env, cwd=root, timeout=600)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


def test_async_calls_on_different_torch_streams_share_scratch_safely():
    """Device entry points run on torch's current stream; a context's scratch
    (Gram panel, series row sums) is shared, so switching streams orders the
    new stream after the old one's queued work (zk_ctx_set_stream).
    Back-to-back async Gram/series calls on two streams must equal the
    synchronous results."""
    modes = zb.full_mode_set(24)
    rho, theta = disc(50_000, 9)
    r_d = torch.from_numpy(rho).cuda()
    t_d = torch.from_numpy(theta).cuda()
    c = torch.from_numpy(np.random.default_rng(9).standard_normal(len(modes))).cuda()
    ref_f = zb.series_device(modes, c, r_d, t_d).clone()
    ref_G, _ = zb.gram_device(modes, r_d, t_d)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            G1, _ = zb.gram_device(modes, r_d, t_d)
            f1 = zb.series_device(modes, c, r_d, t_d)
        with torch.cuda.stream(s2):
            G2, _ = zb.gram_device(modes, r_d, t_d)
            f2 = zb.series_device(modes, c, r_d, t_d)
        outs += [(G1, f1, s1), (G2, f2, s2)]
    torch.cuda.synchronize()
    for G, f, _ in outs:
        assert torch.equal(G, ref_G) and torch.equal(f, ref_f)


def test_release_buffers_then_recompute():
    """release_buffers() frees the host result pool and every context's
    device scratch / staging ring; the next calls re-allocate transparently."""
    modes = zb.full_mode_set(30)
    grid = zb.linear_radial_grid(20_000)
    a, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=grid))
    av = a.values.copy()
    zb.release_buffers()
    b, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=grid))
    assert np.array_equal(b.values, av)


def test_series_and_gram_empty_and_single_mode_edges():
    """Degenerate shapes through the numpy API: no points (f has shape (0,) /
    (0, V), G = 0), one mode (M = 1, the Gram's 1 x 1 block inside a 64-wide
    tile), and a single point."""
    modes = zb.full_mode_set(6)
    M = len(modes)
    f = zb.series_eval(modes, np.ones((M, 3)), np.zeros(0), np.zeros(0))
    assert f.shape == (0, 3)
    G, r = zb.gram(modes, np.zeros(0), np.zeros(0), np.zeros(0))
    assert G.shape == (M, M) and not np.any(np.asarray(G.cpu() if hasattr(G, "cpu") else G))
    one = zb.as_mode_set([(4, -2)])
    rho, theta = disc(301, 77)
    B = orc.basis_2d([(4, -2)], rho, theta)
    f = zb.series_eval(one, np.array([2.5]), rho, theta)
    assert np.abs(f - 2.5 * B[:, 0]).max() <= 1e-13
    G, r = zb.gram(one, rho, theta, f)
    G = np.asarray(G.cpu() if hasattr(G, "cpu") else G)
    r = np.asarray(r.cpu() if hasattr(r, "cpu") else r)
    assert abs(G[0, 0] - B[:, 0] @ B[:, 0]) <= 1e-12 * (B[:, 0] @ B[:, 0])
    assert abs(r[0] - B[:, 0] @ f) <= 1e-12 * abs(B[:, 0]) @ abs(f)
    rho1, theta1 = disc(1, 5)
    f1 = zb.series_eval(modes, np.arange(M, dtype=float), rho1, theta1)
    B1 = orc.basis_2d([(md.n, md.m) for md in modes], rho1, theta1)
    assert np.abs(f1 - B1 @ np.arange(M)).max() <= 1e-12 * np.abs(B1).sum() * M


@pytest.mark.parametrize("seed", range(12))
def test_series_random_requests_against_oracle(seed):
    """Seeded random requests through every series engine the dispatcher picks:
    random mode lists (duplicates, sign flips, sparse alpha), 1..10 vectors,
    derivative order 0..3, 2-D or radial, point counts that are not tile
    multiples; every entry against B @ C of the oracle."""
    rng = np.random.default_rng(1000 + seed)
    nmax = int(rng.integers(1, 40))
    pool = [(n, m) for n in range(nmax + 1) for m in range(-n, n + 1, 2)]
    M = int(rng.integers(1, min(len(pool), 120) + 1))
    pairs_ = [pool[i] for i in rng.integers(0, len(pool), size=M)]
    modes = zb.as_mode_set(pairs_)
    V = int(rng.integers(1, 11))
    k = int(rng.integers(0, 4))
    P = int(rng.integers(1, 2500))
    rho, theta = disc(P, seed)
    two_d = bool(rng.integers(0, 2))
    C = rng.standard_normal((M, V))
    f = zb.series_eval(modes, C, rho, theta if two_d else None, k)
    B = orc.basis_2d(pairs_, rho, theta, k) if two_d else orc.radial_batch(pairs_, rho, k)
    scale = np.abs(B) @ np.abs(C)
    err = np.abs(f.reshape(P, V) - B @ C)
    assert (err <= 1e-12 * scale + 1e-300).all(), (seed, M, V, k, P, two_d, float(err.max()))


@pytest.mark.parametrize("seed", range(8))
def test_gram_random_requests_against_numpy(monkeypatch, seed):
    """Seeded random normal-equation requests: random mode lists (so M + 1 hits
    every residue mod the 64-column block), 2-D or radial, point counts that
    are not multiples of the 16-point step, one or several panels; G and B^T y
    against numpy on the oracle basis, G exactly symmetric."""
    rng = np.random.default_rng(2000 + seed)
    nmax = int(rng.integers(1, 30))
    pool = [(n, m) for n in range(nmax + 1) for m in range(-n, n + 1, 2)]
    M = int(rng.integers(1, min(len(pool), 200) + 1))
    pairs_ = [pool[i] for i in rng.integers(0, len(pool), size=M)]
    modes = zb.as_mode_set(pairs_)
    P = int(rng.integers(1, 6000))
    rho, theta = disc(P, 50 + seed)
    two_d = bool(rng.integers(0, 2))
    y = rng.standard_normal(P)
    if seed % 2:
        monkeypatch.setenv("ZK_GRAM_PANEL_MB", "1")  # several panels
    G, r = zb.gram(modes, rho, theta if two_d else None, y)
    G = np.asarray(G.cpu() if hasattr(G, "cpu") else G)
    r = np.asarray(r.cpu() if hasattr(r, "cpu") else r)
    B = orc.basis_2d(pairs_, rho, theta) if two_d else orc.radial_batch(pairs_, rho, 0)
    gs = np.abs(B).T @ np.abs(B)
    assert (np.abs(G - B.T @ B) <= 1e-12 * gs + 1e-300).all(), (seed, M, P, two_d)
    assert np.array_equal(G, G.T)
    assert (np.abs(r - B.T @ y) <= 1e-12 * (np.abs(B).T @ np.abs(y)) + 1e-300).all()


def test_series_high_alpha_terms_accuracy_vs_binary128(monkeypatch):
    """A mode set of high |m| only (the terms whose rho^|m| e^{i|m|theta} the
    resident kernel advances by complex multiplies between anchors), against
    the binary128 oracle: error per point relative to sum |B||c|, no worse than
    twice the exact-arithmetic engine's (measured: 1.028e-14 vs 1.026e-14 --
    the same whether the kernel re-anchors every 8, 32 or no alpha-steps)."""
    pairs_ = [(n, m) for n in range(40, 61) for m in range(-n, n + 1, 2) if abs(m) >= 40]
    modes = zb.as_mode_set(pairs_)
    rho, theta = disc(2000, 61)
    rho = np.sqrt(rho)  # push points toward the rim, where rho^|m| is not small
    c = np.random.default_rng(62).standard_normal(len(pairs_))
    Bq = orc.quad_table(pairs_, rho, 0)
    m = np.array([p[1] for p in pairs_])
    ang = np.where(m >= 0, np.cos(np.abs(m)[None, :] * theta[:, None]),
                   np.sin(np.abs(m)[None, :] * theta[:, None]))
    B2 = Bq * ang
    ref = (B2.astype(np.longdouble) @ c.astype(np.longdouble)).astype(np.float64)
    scale = np.abs(B2) @ np.abs(c)
    errs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ZK_SERIES_EXACT", mode)
        f = zb.series_eval(modes, c, rho, theta)
        errs[mode] = float((np.abs(f - ref) / scale).max())
    print(f"high-alpha series error {errs['0']:.3e} (exact engine {errs['1']:.3e}) of sum|B||c|")
    assert errs["0"] <= 2 * errs["1"] + 1e-15


def test_gram_panel_geometries_bitwise(monkeypatch):
    """The Gram is bitwise independent of its panel geometry switches read per
    call: one panel, several double-buffered panels (K2 of panel i+1 overlapping
    the SYRK of panel i), and several panels without the overlap."""
    modes = zb.full_mode_set(20)
    rho, theta = disc(40_000, 71)
    y = np.random.default_rng(72).standard_normal(40_000)
    outs = []
    for env in ({}, {"ZK_GRAM_PANEL_MB": "1"}, {"ZK_GRAM_PANEL_MB": "1", "ZK_GRAM_OVERLAP": "0"}):
        for k in ("ZK_GRAM_PANEL_MB", "ZK_GRAM_OVERLAP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        G, r = zb.gram(modes, rho, theta, y)
        outs.append((np.asarray(G.cpu() if hasattr(G, "cpu") else G),
                     np.asarray(r.cpu() if hasattr(r, "cpu") else r)))
    # the panel split changes the summation order across panels, so one panel
    # vs several is tolerance-equal; the overlap switch alone is bitwise
    assert np.array_equal(outs[1][0], outs[2][0]) and np.array_equal(outs[1][1], outs[2][1])
    B = orc.basis_2d([(md.n, md.m) for md in modes], rho, theta)
    gs = np.abs(B).T @ np.abs(B)
    for G, r in outs:
        assert (np.abs(G - B.T @ B) <= 1e-12 * gs).all()
        assert (np.abs(r - B.T @ y) <= 1e-12 * (np.abs(B).T @ np.abs(y))).all()


@pytest.mark.parametrize("panel_mb", [None, "1"])
def test_gram_accumulate_is_cuda_graph_capturable(monkeypatch, panel_mb):
    """zk_gram_accumulate on device buffers captures into a CUDA graph on the
    caller's stream -- one panel, or several double-buffered panels whose K2
    runs on the library's second stream (joined through events) -- and the
    replay is bitwise the eager call."""
    import torch
    if panel_mb:
        monkeypatch.setenv("ZK_GRAM_PANEL_MB", panel_mb)
    modes = zb.full_mode_set(30)
    n = np.array([md.n for md in modes], np.int32)
    m = np.array([md.m for md in modes], np.int32)
    M, P = n.size, 20_000
    ctx = zb._lib.context(0)
    plan = zb._lib.plan_for(ctx, n, m)
    rng = np.random.default_rng(9)
    rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
    th = torch.from_numpy(rng.uniform(-3, 3, size=P)).cuda()
    y = torch.from_numpy(rng.standard_normal(P)).cuda()
    G = torch.zeros((M, M), dtype=torch.float64, device="cuda")
    r = torch.zeros(M, dtype=torch.float64, device="cuda")

    def call():
        G.zero_()
        r.zero_()
        zb._lib.check(zb._lib.lib.zk_gram_accumulate(ctx.handle, plan.handle, rho.data_ptr(),
                                                     th.data_ptr(), P, y.data_ptr(), G.data_ptr(),
                                                     r.data_ptr(), zb._lib.ZK_ASYNC), "gram")

    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    try:
        with torch.cuda.stream(s):
            call()
        torch.cuda.synchronize()
        eager = (G.clone(), r.clone())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call()
        G.fill_(7.0)
        r.fill_(7.0)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(eager[0], G) and torch.equal(eager[1], r)
    finally:
        ctx.set_stream(None)


def test_concurrent_mixed_entry_points_share_a_context():
    """Host threads mixing the series, the Gram and the 2-D basis on one device
    context (one call at a time per context; the staged host paths share its
    scratch and ring) get the serial results bitwise."""
    from concurrent.futures import ThreadPoolExecutor
    modes = zb.full_mode_set(25)
    n = np.array([md.n for md in modes], np.int32)
    m = np.array([md.m for md in modes], np.int32)
    rho, theta = disc(20_000, 81)
    c = np.random.default_rng(82).standard_normal(len(modes))
    y = np.random.default_rng(83).standard_normal(20_000)
    def gram_g():
        G = zb.gram(modes, rho, theta, y)[0]
        return np.asarray(G.cpu() if hasattr(G, "cpu") else G)

    jobs = [lambda: zb.series_eval(modes, c, rho, theta), gram_g,
            lambda: zb.zernike_basis(rho, theta, n, m)]
    want = [j() for j in jobs]
    with ThreadPoolExecutor(6) as pool:
        got = list(pool.map(lambda i: jobs[i % 3](), range(18)))
    for i, g in enumerate(got):
        assert np.array_equal(g, want[i % 3]), i


def test_solve_normal_rejects_an_indefinite_normal_matrix():
    """K6 raises torch.linalg.LinAlgError (as torch.linalg.cholesky would) when
    the matrix is not positive definite, and a duplicated mode (two equal
    columns of B: singular G) solves once regularised."""
    import torch
    modes = zb.as_mode_set([(2, 0), (2, 0), (4, 2)])
    rho, theta = disc(500, 91)
    y = np.random.default_rng(92).standard_normal(500)
    G, r = zb.gram(modes, rho, theta, y)
    G = torch.as_tensor(G, device="cuda")
    with pytest.raises(torch.linalg.LinAlgError):
        zb.solve_normal(-G, r)
    x = zb.solve_normal(G, r, ridge=1e-9 * float(G.diagonal().max()))
    assert torch.isfinite(x).all()


@pytest.mark.parametrize("two_d", [True, False])
def test_emulated_gram_matches_dmma(monkeypatch, two_d):
    """The opt-in fp64-emulated Gram (ZK_GRAM_EMULATED=1: int8 slices, tcgen05
    int8 GEMMs from the CuTe-DSL library kernel, fp64 recombination) against
    the DMMA Gram on the same points: within 1e-13 of |B|^T|B|; several point
    chunks (P > 524,160) and a mode count that is not a multiple of the
    256-row tile. Skipped when the CuTe-DSL GEMM is not installed."""
    import torch
    try:
        from paper_2409_19156_b200 import gram_emulated as ge
        ge._example_module()
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"CuTe-DSL GEMM unavailable: {exc}")
    modes = zb.full_mode_set(24)
    P = 600_001
    rng = np.random.default_rng(101)
    rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
    th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda() if two_d else None
    y = torch.from_numpy(rng.standard_normal(P)).cuda()
    G0, r0 = zb.gram_device(modes, rho, th, y)
    monkeypatch.setenv("ZK_GRAM_EMULATED", "1")
    G1, r1 = zb.gram_device(modes, rho, th, y)
    B = zb.basis_device(modes, rho, theta=th)
    aB = B.abs()
    scale = aB.t() @ aB
    rscale = aB.t() @ y.abs()
    assert float(((G1 - G0).abs() / scale).max()) <= 1e-13
    assert float(((r1 - r0).abs() / rscale).max()) <= 1e-13
    assert torch.equal(G1, G1.t())
