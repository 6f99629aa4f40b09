"""GPU parity of K1 (radial basis, orders 0..3), K2 (2-D basis) and the
chain export against the CPU oracle and the reference's golden vectors.
Every call goes through the C ABI (libzk_b200.so)."""

import ctypes

import numpy as np
import pytest

import zk_oracle as orc
from conftest import rel_err, within_tolerance

pytestmark = pytest.mark.gpu

zb = pytest.importorskip("paper_2409_19156_b200")
from paper_2409_19156_b200 import _lib  # noqa: E402


def pairs(modes):
    return [(md.n, md.m) for md in modes]


def radial(modes, grid, k=0):
    t, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=grid, deriv_order=k))
    return t.values


# --------------------------------------------------------------------------
# configs vs oracle / golden
# --------------------------------------------------------------------------

@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_config1_matches_oracle_and_golden(golden, k):
    modes = zb.full_mode_set(20)
    grid = golden["c1_grid_k0"] if k == 0 else golden["c1_grid_k123"]
    got = radial(modes, grid, k)
    ref = orc.radial_batch(pairs(modes), grid, k)
    assert within_tolerance(got, ref)
    assert rel_err(got[:, golden["c1_ucols"]], golden[f"c1_k{k}"]) <= 1e-12
    # m = 0 columns use no power of rho for k = 0: the recursion is bitwise
    # the reference's (exact division via the Markstein correction)
    if k == 0:
        m0 = [c for c, md in enumerate(modes) if md.m == 0]
        assert np.array_equal(got[:, m0], ref[:, m0])


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_config2_subsample_matches_golden(golden, k):
    modes = zb.full_mode_set(100)
    grid = golden["c2_grid"] if k == 0 else golden["c2_grid"][::4]
    got = radial(modes, grid, k)[:, golden["c2_ucols"]]
    assert within_tolerance(got, golden[f"c2_k{k}"])
    # most entries are bitwise the reference's (only rho**m can differ)
    assert np.mean(got == golden[f"c2_k{k}"]) > 0.5


def test_config2_full_size_spot_checks():
    """n=100 x 1e5 (config 2) through the numpy API; every point is
    independent, so a seeded subsample is checked against the oracle."""
    modes = zb.full_mode_set(100)
    grid = zb.linear_radial_grid(100_000)
    got = radial(modes, grid, 0)
    assert got.shape == (100_000, 5151) and got.flags.f_contiguous
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([[0, 1, 99_999], rng.integers(0, 100_000, 61)]))
    ref = orc.radial_batch(pairs(modes), grid[idx], 0)
    assert within_tolerance(got[idx], ref)
    # R_n^m(1) = 1 for every mode (reference tests/test_evaluate.py:114-117)
    assert np.abs(got[-1] - 1.0).max() <= 1e-11
    # centre values (tests/test_evaluate.py:86-91)
    want0 = np.array([0.0 if md.m else (1.0 if md.n % 4 == 0 else -1.0) for md in modes])
    assert np.abs(got[0] - want0).max() <= 1e-15


def test_config3_all_orders_equal_single_order_bitwise():
    modes = zb.full_mode_set(100)
    grid = zb.linear_radial_grid(20_000)
    req = zb.BatchRequest(modes=modes, grid=grid, deriv_order=3)
    mats = zb.evaluate_batch_all_orders(req)
    assert [m.deriv_order for m in mats] == [0, 1, 2, 3]
    for k in range(4):
        single = radial(modes, grid, k)
        assert np.array_equal(mats[k].values, single), k
    rng = np.random.default_rng(1)
    idx = rng.integers(0, grid.size, 24)
    for k in range(4):
        ref = orc.radial_batch(pairs(modes), grid[idx], k)
        assert within_tolerance(mats[k].values[idx], ref), k


def test_config4_high_order_error_no_worse_than_reference(golden):
    """n=200 (20,301 modes) x 1e4: max-abs error against the exact bigint
    oracle must not exceed the reference's own error on the same points."""
    modes = zb.full_mode_set(200)
    P = 10_000
    grid = zb.linear_radial_grid(P)
    got = radial(modes, grid, 0)
    ucols = golden["c4_ucols"]
    rng = np.random.default_rng(2)
    idx = np.unique(np.concatenate([[0, 1, P // 3, P - 2, P - 1], rng.integers(0, P, 19)]))
    pts = grid[idx]
    umodes = [pairs(modes)[c] for c in ucols]
    exact = orc.exact_table(umodes, pts, 0)
    ref = orc.radial_batch(umodes, pts, 0)
    err_gpu = np.abs(got[idx][:, ucols] - exact).max()
    err_ref = np.abs(ref - exact).max()
    assert err_gpu <= err_ref, (err_gpu, err_ref)
    # and on the committed golden points (exact oracle from the reference)
    gidx = np.searchsorted(grid, golden["c4_grid"])
    assert np.array_equal(grid[gidx], golden["c4_grid"])
    err_gpu_g = np.abs(got[gidx][:, ucols] - golden["c4_exact"]).max()
    err_ref_g = np.abs(golden["c4_k0"] - golden["c4_exact"]).max()
    assert err_gpu_g <= err_ref_g, (err_gpu_g, err_ref_g)


def test_config4_full_grid_error_vs_binary128_oracle():
    """The n=200 clause at scale: every mode on every 5th point of the 1e4-point
    grid (2,000 points x 20,301 columns), max-abs error against the binary128
    oracle (bitwise equal to the exact oracle, tests/test_oracle.py) is no worse
    than the reference algorithm's own error on the same entries."""
    modes = zb.full_mode_set(200)
    grid = zb.linear_radial_grid(10_000)
    got = radial(modes, grid, 0)[::5]
    pts = grid[::5]
    umodes = [(n, a) for n in range(201) for a in range(n % 2, n + 1, 2)]
    ucols = [c for c, md in enumerate(modes) if md.m >= 0]
    exact = orc.quad_table(umodes, pts, 0)
    ref = orc.radial_batch(umodes, pts, 0)
    err_gpu = float(np.abs(got[:, ucols] - exact).max())
    err_ref = float(np.abs(ref - exact).max())
    print(f"n<=200, 2000 pts: max-abs error gpu {err_gpu:.3e}, reference {err_ref:.3e}")
    assert err_gpu <= err_ref, (err_gpu, err_ref)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_config2_3_error_vs_binary128_oracle(k):
    """n<=100 on 500 points of the config-2 grid, every order: GPU error vs the
    exact value within the north_star tolerance, and on par with the
    reference algorithm's own error."""
    modes = [(n, a) for n in range(101) for a in range(n % 2, n + 1, 2)]
    grid = zb.linear_radial_grid(100_000)[::200]
    got = radial(zb.as_mode_set(modes), grid, k)
    exact = orc.quad_table(modes, grid, k)
    ref = orc.radial_batch(modes, grid, k)
    scale = np.maximum(1.0, np.abs(exact).max(axis=0))
    e_gpu = float((np.abs(got - exact).max(axis=0) / scale).max())
    e_ref = float((np.abs(ref - exact).max(axis=0) / scale).max())
    print(f"k={k}: relative error gpu {e_gpu:.3e}, reference {e_ref:.3e}")
    assert e_gpu <= 1e-12
    assert e_gpu <= 2 * e_ref + 1e-15


def test_config5_2d_basis_matches_golden(golden):
    modes = zb.full_mode_set(60)
    n = np.array([md.n for md in modes])
    m = np.array([md.m for md in modes])
    B = zb.zernike_basis(golden["c5_rho"], golden["c5_theta"], n, m)
    assert within_tolerance(B, golden["c5_B"])
    for k in (1, 2, 3):
        Bk = zb.zernike_basis(golden["c5_rho"], golden["c5_theta"], n, m, k)
        assert within_tolerance(Bk, golden[f"c5_B_k{k}"]), k
    f = B @ golden["c5_coef"]
    assert np.abs(f - golden["c5_f"]).max() <= 1e-11


# --------------------------------------------------------------------------
# the reference's cross-entry-point bitwise invariants
# --------------------------------------------------------------------------

def test_batch_column_equals_single_mode_call():
    grid = zb.linear_radial_grid(37)
    modes = zb.full_mode_set(10)
    table = radial(modes, grid, 2)
    for col, md in enumerate(modes):
        assert np.array_equal(table[:, col], zb.radial_jacobi(md.n, md.m_abs, grid, 2))


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_strategies_agree_bitwise(k):
    grid = zb.linear_radial_grid(100)
    modes = zb.full_mode_set(12)
    a, ca = zb.batch_cached(zb.BatchRequest(modes=modes, grid=grid, deriv_order=k))
    b, cb = zb.batch_independent(
        zb.BatchRequest(modes=modes, grid=grid, deriv_order=k, strategy="independent"))
    assert np.array_equal(a.values, b.values)
    assert ca.recursion_steps <= cb.recursion_steps and ca.chain_count <= cb.chain_count
    s, _ = zb.batch_cached(zb.BatchRequest(modes=modes, grid=grid, deriv_order=k), parallel=True)
    assert np.array_equal(a.values, s.values)


def test_duplicate_and_sign_flipped_columns():
    grid = zb.linear_radial_grid(21)
    modes = zb.as_mode_set([(4, 2), (4, -2), (4, 2), (2, 0), (4, 2)])
    table, counter = zb.batch_cached(zb.BatchRequest(modes=modes, grid=grid))
    for c in (1, 2, 4):
        assert np.array_equal(table.values[:, 0], table.values[:, c])
    assert counter.chain_count == 2


def test_arbitrary_requests_match_oracle(golden):
    for r in range(6):
        modes = zb.as_mode_set([tuple(x) for x in golden[f"idx_req{r}"].tolist()])
        for k in (0, 2):
            got = radial(modes, golden["idx_req_grid"], k)
            assert within_tolerance(got, golden[f"idx_req{r}_k{k}"]), (r, k)


def test_zernike_eval_angular_split_is_exact():
    rho = np.array([0.6])
    for n, m in [(3, 1), (4, 2), (5, 3)]:
        radial1 = zb.radial_jacobi(n, m, rho)[0]
        assert zb.zernike_eval(zb.make_mode(n, m), rho, [0.0])[0] == radial1
        assert zb.zernike_eval(zb.make_mode(n, -m), rho, [0.0])[0] == 0.0
        q = np.pi / (2 * m)
        assert zb.zernike_eval(zb.make_mode(n, -m), rho, [q])[0] == pytest.approx(radial1, rel=1e-12)
    assert zb.zernike_eval(zb.make_mode(2, 2), [1.0], [0.0])[0] == pytest.approx(1.0, abs=1e-14)
    assert zb.zernike_eval(zb.make_mode(1, 1), [0.5], [np.pi])[0] == pytest.approx(-0.5, abs=1e-15)
    assert zb.zernike_eval(zb.make_mode(2, 0), [0.5], [1.234], 1)[0] == pytest.approx(2.0, abs=1e-14)


def test_zernike_eval_equals_oracle_per_mode():
    rng = np.random.default_rng(3)
    rho = rng.uniform(size=33)
    th = rng.uniform(-7, 7, size=33)
    for md in zb.full_mode_set(16):
        for k in (0, 3):
            got = zb.zernike_eval(md, rho, th, k)
            ref = orc.zernike_2d(md.n, md.m, rho, th, k)
            assert within_tolerance(got[:, None], ref[:, None]), (md, k)


# --------------------------------------------------------------------------
# known answers of the reference tests
# --------------------------------------------------------------------------

def test_exact_zero_and_constant_derivatives():
    grid = np.linspace(0.0, 1.0, 7)
    for k in (1, 2, 3):
        assert np.all(zb.radial_jacobi(0, 0, grid, k) == 0.0)
    assert np.all(zb.radial_jacobi(1, 1, grid, 2) == 0.0)
    assert np.all(zb.radial_jacobi(2, 2, grid, 3) == 0.0)
    assert np.all(zb.radial_jacobi(3, 3, grid, 3) == 6.0)
    assert zb.radial_jacobi(1, 1, [0.3])[0] == pytest.approx(0.3, abs=1e-15)
    assert zb.radial_jacobi(2, 0, [0.5])[0] == pytest.approx(-0.5, abs=1e-15)
    assert zb.radial_jacobi(4, 0, [1.0])[0] == pytest.approx(1.0, abs=1e-14)
    assert zb.radial_jacobi(2, 0, [0.5], 1)[0] == pytest.approx(2.0, abs=1e-14)
    assert zb.radial_jacobi(0, 0, [0.0])[0] == 1.0  # 0**0 == 1


def test_endpoint_is_one_to_n150():
    modes = [zb.make_mode(n, m) for n in range(0, 151, 7) for m in range(n % 2, n + 1, 2)]
    got = radial(modes, [1.0])
    assert np.abs(got - 1.0).max() <= 1e-11


def test_finite_difference_first_derivative():
    h = 1e-6
    pts = np.linspace(0.1, 0.9, 33)
    modes = [zb.make_mode(n, m) for n in range(31) for m in range(n % 2, n + 1, 2)]
    d1 = radial(modes, pts, 1)
    fd = (radial(modes, pts + h) - radial(modes, pts - h)) / (2 * h)
    scale = np.maximum(1.0, np.abs(d1).max(axis=0))
    assert (np.abs(fd - d1).max(axis=0) / scale).max() < 1e-4


def test_low_order_modes_match_exact_oracle():
    # tests/test_evaluate.py:93-101: n <= 12, every order, 1e-12 relative
    from fractions import Fraction
    grid = zb.linear_radial_grid(100)
    modes = [(n, m) for n in range(13) for m in range(n % 2, n + 1, 2)]
    for k in range(4):
        exact = orc.exact_table(modes, grid, k)
        got = radial(zb.as_mode_set(modes), grid, k)
        assert rel_err(got, exact) <= 1e-12, k
    assert Fraction(grid[3]) == Fraction(grid[3])


def test_jacobi_chain_bitwise_and_scipy():
    from scipy.special import eval_jacobi
    x = np.linspace(-1.0, 1.0, 23)
    for a, b in [(0, 0), (1, 0), (5, 0), (2, 2), (7, 3)]:
        got = zb.jacobi_chain(12, a, b, x)
        assert np.array_equal(got, orc.jacobi_chain(12, a, b, x))
        for d in range(13):
            want = eval_jacobi(d, a, b, x)
            assert (np.abs(got[d] - want) / np.maximum(1.0, np.abs(want))).max() < 1e-12
    assert np.all(zb.jacobi_chain(0, 3, 1, x)[0] == 1.0)
    assert zb.jacobi_chain(1, 2, 0, [-1.0])[1][0] == -1.0
    assert zb.jacobi_chain(2, 0, 0, [0.5])[2][0] == -0.125


# --------------------------------------------------------------------------
# C ABI paths: device buffers, ld > P, odd P, scalar vs vector stores,
# host-in/device-out, multi-chunk host-out pipeline
# --------------------------------------------------------------------------

torch = pytest.importorskip("torch")


def _plan(modes):
    ctx = _lib.context()
    n = np.array([md.n for md in modes], np.int32)
    m = np.array([md.m for md in modes], np.int32)
    return ctx, _lib.plan_for(ctx, n, m)


@pytest.mark.parametrize("P", [1, 2, 255, 256, 257, 1001])
def test_device_paths_ld_and_tails(P):
    modes = zb.full_mode_set(9)
    M = len(modes)
    ctx, plan = _plan(modes)
    grid = np.random.default_rng(P).uniform(size=P)
    ref = radial(modes, grid, 2)
    d_rho = torch.tensor(grid, device="cuda")
    for ld, flags in [(P, 0), (P + 3, 0), (P + (P % 2), _lib.ZK_STORE_SCALAR), (P + 8, 0)]:
        out = torch.full((M, ld), float("nan"), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, d_rho.data_ptr(), P, 2, 0,
                                           out.data_ptr(), ld, 0, flags), "radial")
        host = out.cpu().numpy()
        assert np.array_equal(host[:, :P].T, ref), (ld, flags)
        assert np.isnan(host[:, P:]).all()  # padding untouched


def test_host_input_device_output_and_all_orders_stride():
    modes = zb.full_mode_set(14)
    M, P = len(modes), 3000
    ctx, plan = _plan(modes)
    grid = zb.linear_radial_grid(P)
    ld, ostride = P + 2, (P + 2) * M + 64
    out = torch.zeros(4 * ostride, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, grid.ctypes.data, P, 3, 1,
                                       out.data_ptr(), ld, ostride, _lib.ZK_HOST_INPUT), "radial")
    host = out.cpu().numpy()
    for k in range(4):
        blk = host[k * ostride:k * ostride + ld * M].reshape(M, ld).T[:P]
        assert np.array_equal(blk, radial(modes, grid, k)), k


def test_multi_chunk_host_pipeline_matches_device():
    modes = zb.full_mode_set(100)  # 5151 columns -> ~6.5k points per 256 MB chunk
    P = 40_001
    grid = np.random.default_rng(4).uniform(size=P)
    host = radial(modes, grid, 0)  # chunked D2H path
    ctx, plan = _plan(modes)
    d_rho = torch.tensor(grid, device="cuda")
    out = torch.empty((len(modes), P), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, d_rho.data_ptr(), P, 0, 0,
                                       out.data_ptr(), P, 0, 0), "radial")
    assert np.array_equal(out.cpu().numpy().T, host)


def test_launch_counter_and_errors():
    modes = zb.full_mode_set(4)
    ctx, plan = _plan(modes)
    before = ctx.launches()
    radial(modes, [0.1, 0.2], 1)
    assert ctx.launches() > before
    d = torch.zeros(16, dtype=torch.float64, device="cuda")
    rc = _lib.lib.zk_radial_eval(ctx.handle, plan.handle, d.data_ptr(), 2, 4, 0, d.data_ptr(), 2,
                                 0, 0)
    assert rc == _lib.ZK_EINVAL
    rc = _lib.lib.zk_radial_eval(ctx.handle, plan.handle, d.data_ptr(), 4, 0, 0, d.data_ptr(), 2,
                                 0, 0)
    assert rc == _lib.ZK_EINVAL  # ld < P
    cnt = ctypes.c_int(0)
    assert _lib.lib.zk_device_count(ctypes.byref(cnt)) == 0 and cnt.value >= 1


def test_heavily_duplicated_group_is_split():
    # > 4096 columns with the same |m|: the planner splits the alpha group into
    # virtual groups (shared-memory offset tables stay bounded)
    pairs = [(2, 0)] * 5000 + [(6, 2), (6, -2)] * 1500 + [(4, 0)] * 300
    modes = zb.as_mode_set(pairs)
    grid = np.random.default_rng(11).uniform(size=300)
    ctx, plan = _plan(modes)
    info = plan.info()
    assert info["U"] == 3 and info["groups"] >= 3
    got = radial(modes, grid, 1)
    ref = orc.radial_batch(pairs, grid, 1)
    assert within_tolerance(got, ref)
    assert np.array_equal(got[:, 0], got[:, 4999])


def test_high_degree_sparse_request():
    """Degrees far beyond the configs (n up to 1000, jacobi degree 500): the
    shared-memory coefficient stage scales with jmax; values follow the
    reference algorithm (bitwise recursion) and the binary128 oracle."""
    pairs = [(1000, 0), (1000, 2), (999, 999), (998, -4), (601, 11), (500, 500), (2, 2)]
    modes = zb.as_mode_set(pairs)
    grid = np.concatenate([[0.0, 1.0], np.random.default_rng(12).uniform(size=50)])
    for k in (0, 2):
        got = radial(modes, grid, k)
        ref = orc.radial_batch(pairs, grid, k)
        exact = orc.quad_table(pairs, grid, k)
        err_gpu = np.abs(got - exact).max(axis=0)
        err_ref = np.abs(ref - exact).max(axis=0)
        assert (err_gpu <= 2 * err_ref + 1e-12 * np.maximum(1, np.abs(exact).max(axis=0))).all(), k


def test_concurrent_callers_share_a_context():
    """The reference drives this path from thread pools (zk/batch.py:136-138):
    concurrent calls on one context serialise safely and agree bitwise."""
    from concurrent.futures import ThreadPoolExecutor
    modes = zb.full_mode_set(30)
    grid = zb.linear_radial_grid(777)
    want = radial(modes, grid, 1)
    with ThreadPoolExecutor(8) as pool:
        outs = list(pool.map(lambda _: radial(modes, grid, 1), range(16)))
    for o in outs:
        assert np.array_equal(o, want)


def test_degree_6000_uses_the_global_coefficient_kernel():
    # jacobi degree 3000 with k=3 cannot stage its coefficients in shared
    # memory (it used to fail with ValueError); the fallback kernel serves it
    modes = zb.as_mode_set([(6000, 0), (5999, 1)])
    pts = np.array([0.0, 0.25, 0.5, 0.999, 1.0])
    got = radial(modes, pts, 3)
    want = orc.radial_batch([(6000, 0), (5999, 1)], pts, 3, power=orc.cr_power)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_subnormal_rho_powers(k):
    """Where rho^(|m|+k) < 2^-916 the double-double power window's error terms
    underflow, so the bitwise claim (the reference algorithm with correctly
    rounded powers) covers only entries whose window stays above that; below,
    the power is within a few subnormal ulps -- inside the parity tolerance,
    and numpy's own pow (the reference) is not correctly rounded there either.
    High-degree cases (values ~1e-200 from subnormal powers times huge chains)
    found by tools/fuzz_paths.py seed 777; DESIGN.md section 3."""
    from fractions import Fraction
    pairs_ = [(2008, -1876), (2281, -483), (2031, 1071), (1928, 1778), (2515, -703),
              (400, 380), (600, 560), (40, 12)]
    modes = zb.as_mode_set(pairs_)
    pts = np.array([0.6810649396839922, 0.6629706704580528, 0.50270979, 0.82940846,
                    0.02, 0.15, 0.3, 1e-160, 0.0])
    got = radial(modes, pts, k)
    want = orc.radial_batch([(md.n, md.m) for md in modes], pts, k, power=orc.cr_power)
    exact = np.array([[float(Fraction(float(r)) ** (abs(md.m) + k)) >= 2.0 ** -916
                       for md in modes] for r in pts])
    fin = np.isfinite(want)
    assert (exact & fin).sum() > 20 and (~exact & fin & (np.abs(want) > 1e-250)).sum() > 0
    assert np.array_equal(got[exact], want[exact], equal_nan=True)
    assert np.array_equal(np.isfinite(got), fin)
    err = np.abs(np.where(fin, got - want, 0.0))
    assert (err <= 1e-13 + 1e-12 * np.abs(np.where(fin, want, 0.0))).all()


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_exact_power_mode_is_bitwise_everywhere(monkeypatch, k):
    """The opt-in exact-power mode (ZK_EXACT_POW / the C-ABI flag
    ZK_EXACT_POW): powers carried as (double-double mantissa, binary
    exponent) and rounded once, subnormals included -- the reference
    algorithm with correctly rounded powers reproduces EVERY entry bitwise,
    also the ones test_subnormal_rho_powers exempts; above the bound the two
    modes agree bit for bit."""
    pairs_ = [(2008, -1876), (2281, -483), (2031, 1071), (1928, 1778), (2515, -703),
              (400, 380), (600, 560), (40, 12), (100, 100), (100, 60)]
    modes = zb.as_mode_set(pairs_)
    pts = np.array([0.6810649396839922, 0.6629706704580528, 0.50270979, 0.82940846,
                    0.02, 0.15, 0.3, 1e-160, 1e-5, 2e-5, 3e-300, 0.0])
    fast = radial(modes, pts, k)
    monkeypatch.setenv("ZK_EXACT_POW", "1")
    got = radial(modes, pts, k)
    want = orc.radial_batch([(md.n, md.m) for md in modes], pts, k, power=orc.cr_power)
    assert np.array_equal(got, want, equal_nan=True)
    from fractions import Fraction
    normal = np.array([[float(Fraction(float(r)) ** (abs(md.m) + k)) >= 2.0 ** -916
                        for md in modes] for r in pts])
    assert np.array_equal(got[normal], fast[normal], equal_nan=True)
    # the all-orders sweep in exact mode equals the single-order launches
    mats = zb.evaluate_batch_all_orders(zb.BatchRequest(modes=modes, grid=pts, deriv_order=k))
    assert np.array_equal(mats[k].values, got, equal_nan=True)


@pytest.mark.parametrize("vec", ["4", "2", "1"])
def test_store_paths_agree_bitwise(monkeypatch, vec):
    """Every store path (32/16/8-byte direct stores; the TMA bulk-store ring
    staged through shared memory) writes the same bits, including partial
    tiles, all-orders strides and the 2-D basis."""
    modes = zb.full_mode_set(40)
    grid = np.random.default_rng(13).uniform(size=5003)  # partial last tile
    th = np.random.default_rng(14).uniform(-3, 3, size=5003)
    n = np.array([md.n for md in modes])
    m = np.array([md.m for md in modes])
    monkeypatch.setenv("ZK_VEC", vec)
    monkeypatch.setenv("ZK_TMA", "0")
    base = zb.evaluate_batch_all_orders(zb.BatchRequest(modes=modes, grid=grid, deriv_order=3))
    base2d = zb.zernike_basis(grid, th, n, m)
    monkeypatch.setenv("ZK_TMA", "1")
    tma = zb.evaluate_batch_all_orders(zb.BatchRequest(modes=modes, grid=grid, deriv_order=3))
    tma2d = zb.zernike_basis(grid, th, n, m)
    for a, b in zip(base, tma):
        assert np.array_equal(a.values, b.values)
    assert np.array_equal(base2d, tma2d)
    ref = orc.radial_batch(pairs(modes), grid[:64], 3)
    assert within_tolerance(base[3].values[:64], ref)


def test_single_order_cta_sizes_agree_bitwise(tmp_path):
    """Single-order k >= 2 requests run 128-thread CTAs by default and 256-thread
    ones with ZK_SMALL_CTA=0 (read once per process, hence subprocesses): same
    bits, partial tiles included (3,000 points: an even leading dimension keeps
    2 points per thread, the small-CTA condition), and within tolerance of the
    oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]); "
        "import paper_2409_19156_b200 as zb; "
        "modes = zb.full_mode_set(45); "
        "grid = np.random.default_rng(21).uniform(size=3000); "
        "out = [zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=grid, deriv_order=k))[0].values "
        "for k in (2, 3)]; np.save(sys.argv[2], np.stack(out))")
    outs = []
    for flag in ("1", "0"):
        path = tmp_path / f"cta{flag}.npy"
        subprocess.run([sys.executable, "-c", code, root, str(path)], check=True, timeout=600,
                       env=dict(os.environ, ZK_SMALL_CTA=flag), cwd=root)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
    modes = zb.full_mode_set(45)
    grid = np.random.default_rng(21).uniform(size=3000)
    for i, k in enumerate((2, 3)):
        ref = orc.radial_batch(pairs(modes), grid[:50], k)
        assert within_tolerance(outs[0][i][:50], ref)


@pytest.mark.parametrize("env", [
    {"ZK_STAGED": "0"},                              # round 1's land-in-place + fill pipeline
    {"ZK_STAGED": "0", "ZK_BOUNCE": "0"},            # ... without pinned bounce buffers
    {"ZK_UNIQUE_D2H": "0"},                          # every column over PCIe
    {"ZK_RING_SLOTS": "2", "ZK_RING_MB": "1"},       # tiny staging ring
    {"ZK_IMAGE_MB": "64"},                           # several point chunks of the device image
    {"ZK_HOST_THREADS": "1"},                        # copy-out on the calling thread only
])
def test_host_output_paths_bitwise(monkeypatch, env):
    """Every host-output path (read per call) writes the bits of the default
    staged path, for pageable (fresh numpy) and page-locked destinations,
    radial with repeated keys and 2-D, all orders."""
    modes = zb.full_mode_set(40)
    n = np.array([md.n for md in modes], np.int32)
    m = np.array([md.m for md in modes], np.int32)
    grid = np.random.default_rng(31).uniform(size=30001)
    th = np.random.default_rng(32).uniform(-3, 3, size=30001)
    base = zb.evaluate_batch_all_orders(zb.BatchRequest(modes=modes, grid=grid, deriv_order=2))
    base2d = zb.zernike_basis(grid, th, n, m)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = zb.evaluate_batch_all_orders(zb.BatchRequest(modes=modes, grid=grid, deriv_order=2))
    got2d = zb.zernike_basis(grid, th, n, m)
    for a, b in zip(base, got):
        assert np.array_equal(a.values, b.values)
    assert np.array_equal(base2d, got2d)
    # a page-locked destination through the C ABI
    import ctypes
    ctx = zb._lib.context()
    plan = zb._lib.plan_for(ctx, n, m)
    P, M = grid.size, n.size
    hbuf = ctypes.c_void_p()
    zb._lib.check(zb._lib.lib.zk_host_alloc(8 * P * M, ctypes.byref(hbuf)), "zk_host_alloc")
    try:
        zb._lib.check(zb._lib.lib.zk_radial_eval(
            ctx.handle, plan.handle, grid.ctypes.data, P, 0, 0, hbuf.value, P, 0,
            zb._lib.ZK_HOST_INPUT | zb._lib.ZK_HOST_OUTPUT), "zk_radial_eval")
        view = np.ctypeslib.as_array(ctypes.cast(hbuf.value, ctypes.POINTER(ctypes.c_double)),
                                     shape=(M, P))
        assert np.array_equal(view.T, base[0].values)
        del view
    finally:
        zb._lib.lib.zk_host_free(hbuf)


def test_parallel_shards_over_devices_bitwise(monkeypatch):
    """parallel=True splits the points across devices (here: two shards on
    the one available GPU via ZK_DEVICES=0,0); every shard writes its rows of
    the shared F-ordered result and the values are bitwise the serial ones."""
    modes = zb.full_mode_set(25)
    grid = np.random.default_rng(15).uniform(size=7777)
    req = zb.BatchRequest(modes=modes, grid=grid, deriv_order=2)
    serial, cs = zb.batch_cached(req)
    monkeypatch.setenv("ZK_DEVICES", "0,0,0")
    par, cp = zb.batch_cached(req, parallel=True)
    assert np.array_equal(serial.values, par.values) and cs == cp
    n = np.array([md.n for md in modes])
    m = np.array([md.m for md in modes])
    th = np.random.default_rng(16).uniform(size=7777)
    from paper_2409_19156_b200.evaluate import basis_matrix
    a = basis_matrix(n.astype(np.int32), m.astype(np.int32), grid, 1, theta=th, all_orders=True)
    b = basis_matrix(n.astype(np.int32), m.astype(np.int32), grid, 1, theta=th, all_orders=True,
                     devices=[0, 0])
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("pinned", [False, True])
def test_unique_column_host_output_equals_device_output(pinned):
    """Host outputs of the radial basis carry only the unique (n, |m|) columns
    over PCIe and fill the repeated ones on the host (zk_capi.cu, unique view):
    shuffled, duplicated and sign-flipped modes, several chunks, all orders,
    ld > P, pinned and pageable destinations -- bitwise the device result."""
    import ctypes

    rng = np.random.default_rng(21)
    full = [(md.n, md.m) for md in zb.full_mode_set(60)]
    pick = [full[i] for i in rng.permutation(len(full))[:900]]
    pick += pick[:200] + [(n, -m) for n, m in pick[200:400]]
    modes = zb.as_mode_set(pick)
    M, P, k = len(modes), 70_001, 2
    ld = P + 5
    ostride = ld * M + 3
    ctx, plan = _plan(modes)
    grid = rng.uniform(size=P)
    d_rho = torch.tensor(grid, device="cuda")
    dev = torch.empty((k + 1) * ostride, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, d_rho.data_ptr(), P, k, 1,
                                       dev.data_ptr(), ld, ostride, 0), "radial")
    ref = dev.cpu().numpy()
    nbytes = 8 * (k + 1) * ostride
    if pinned:
        buf = ctypes.c_void_p()
        _lib.check(_lib.lib.zk_host_alloc(nbytes, ctypes.byref(buf)), "zk_host_alloc")
        host = np.ctypeslib.as_array(ctypes.cast(buf.value, ctypes.POINTER(ctypes.c_double)),
                                     shape=((k + 1) * ostride,))
    else:
        host = np.empty((k + 1) * ostride)
    host[:] = np.nan
    _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, grid.ctypes.data, P, k, 1,
                                       host.ctypes.data, ld, ostride,
                                       _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT), "radial")
    for o in range(k + 1):
        a = ref[o * ostride:o * ostride + ld * M].reshape(M, ld)[:, :P]
        b = host[o * ostride:o * ostride + ld * M].reshape(M, ld)
        assert np.array_equal(a, b[:, :P]), o
        assert np.isnan(b[:, P:]).all()  # row padding untouched
    if pinned:
        del host
        _lib.lib.zk_host_free(buf)


def test_orthogonality_on_gauss_legendre_nodes():
    """The reference's acceptance criterion 6 (tests/test_acceptance.py:150-172)
    on the GPU basis: for every m, the radial polynomials n, n' <= 40 are
    orthogonal under int_0^1 R_n^m R_n'^m rho drho = delta / (2n + 2), by
    512-node Gauss-Legendre quadrature, to 1e-10."""
    x, w = np.polynomial.legendre.leggauss(512)
    nodes, weights = (x + 1.0) / 2.0, w / 2.0
    modes = zb.as_mode_set([(n, m) for n in range(41) for m in range(n % 2, n + 1, 2)])
    table, _ = zb.batch_cached(zb.BatchRequest(modes=modes, grid=nodes))
    weighted = weights * nodes
    worst = 0.0
    for m in range(41):
        cols = [c for c, md in enumerate(modes) if md.m == m]
        deg = np.array([modes[c].n for c in cols])
        blk = table.values[:, cols]
        gram = blk.T @ (weighted[:, None] * blk)
        worst = max(worst, float(np.abs(gram - np.diag(1.0 / (2.0 * deg + 2.0))).max()))
    assert worst <= 1e-10, worst


def test_basis_device_stays_on_device_and_matches_numpy_path():
    """Device-resident basis: torch tensors in, column-major
    CUDA tensors out, orders 0..k from one sweep; bitwise the numpy path."""
    modes = zb.full_mode_set(30)
    rng = np.random.default_rng(33)
    rho = rng.uniform(size=5000)
    theta = 2 * np.pi * rng.uniform(size=5000)
    d_rho = torch.tensor(rho, device="cuda")
    d_th = torch.tensor(theta, device="cuda")
    B = zb.basis_device(modes, d_rho, 2)
    assert B.is_cuda and B.shape == (5000, len(modes)) and B.stride() == (1, 5000)
    t, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=rho, deriv_order=2))
    assert np.array_equal(B.cpu().numpy(), t.values)
    allo = zb.basis_device(modes, d_rho, 3, all_orders=True)
    assert len(allo) == 4
    for k, Bk in enumerate(allo):
        tk, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=rho, deriv_order=k))
        assert np.array_equal(Bk.cpu().numpy(), tk.values), k
    Z = zb.basis_device(modes, d_rho, 0, theta=d_th)
    for c in (0, 7, len(modes) - 1):
        md = modes[c]
        assert np.array_equal(Z[:, c].cpu().numpy(), zb.zernike_eval(md, rho, theta))
    from torch.utils import dlpack
    again = dlpack.from_dlpack(dlpack.to_dlpack(B))
    assert again.data_ptr() == B.data_ptr()


def test_jacobi_chain_export_matches_reference_golden(golden):
    """zk_jacobi_chain (GPU) == the reference's jacobi_chain, bitwise."""
    x = golden["chain_x"]
    for jm, al, be in golden["chain_cases"]:
        got = zb.jacobi_chain(int(jm), int(al), int(be), x)
        assert np.array_equal(got, golden[f"chain_{jm}_{al}_{be}"]), (jm, al, be)


def test_release_buffers_then_reuse():
    """zk_ctx_release_buffers frees the cached scratch / pinned buffers; the
    next host-output call re-allocates them and gives the same values."""
    modes = zb.full_mode_set(40)
    grid = np.random.default_rng(3).uniform(size=30_000)
    a, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=grid))
    _lib.context().release_buffers()
    b, _ = zb.evaluate_batch(zb.BatchRequest(modes=modes, grid=grid))
    assert np.array_equal(a.values, b.values)


def test_very_long_chains_fall_back_to_global_coefficients():
    """Degrees whose coefficient tables do not fit in shared memory (here
    n = 2500, k = 3: 320 KB) run the global-coefficient fallback kernel --
    still the reference algorithm with correctly rounded powers, bitwise."""
    modes = [(2500, 0), (2500, 2), (2497, 5), (2501, -3), (12, 4)]
    grid = np.random.default_rng(8).uniform(size=300)
    for k in (0, 3):
        t, _ = zb.evaluate_batch(zb.BatchRequest(modes=zb.as_mode_set(modes), grid=grid,
                                                 deriv_order=k))
        want = orc.radial_batch(modes, grid, k, power=orc.cr_power)
        tiny = np.abs(want) < 1e-250
        assert np.array_equal(t.values[~tiny], want[~tiny]), k


@pytest.mark.parametrize("ang", [False, True])
@pytest.mark.parametrize("pinned", [False, True])
def test_small_dense_host_output_equals_device_output(monkeypatch, ang, pinned):
    """Host outputs up to ZK_SMALL_MB take the one-launch / one-D2H path
    (zk_capi.cu eval_common); bitwise the device result and the chunked
    pipeline's, for odd point counts, all orders, the 2-D basis and
    pinned / pageable destinations; ld > P keeps the pipeline."""
    rng = np.random.default_rng(5)
    modes = zb.full_mode_set(30)
    M, k = len(modes), 2
    ctx, plan = _plan(modes)
    for P, extra in ((1, 0), (37, 0), (1001, 0), (1001, 3)):
        ld = P + extra
        ostride = ld * M
        grid = rng.uniform(size=P)
        theta = rng.uniform(0, 2 * np.pi, size=P)
        d_rho = torch.tensor(grid, device="cuda")
        d_th = torch.tensor(theta, device="cuda")
        dev = torch.empty((k + 1) * ostride, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

        def call(rho, th, out, flags):
            if ang:
                return _lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho, th, P, k, 1, out,
                                                ld, ostride, flags)
            return _lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho, P, k, 1, out, ld,
                                           ostride, flags)

        _lib.check(call(d_rho.data_ptr(), d_th.data_ptr(), dev.data_ptr(), 0), "device")
        ref = dev.cpu().numpy()
        flags = _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT
        for small in ("8", "0"):
            monkeypatch.setenv("ZK_SMALL_MB", small)
            if pinned:
                host = torch.full(((k + 1) * ostride,), np.nan, dtype=torch.float64,
                                  pin_memory=True).numpy()
            else:
                host = np.full((k + 1) * ostride, np.nan)
            _lib.check(call(grid.ctypes.data, theta.ctypes.data, host.ctypes.data, flags),
                       "host")
            for o in range(k + 1):
                a = ref[o * ostride:(o + 1) * ostride].reshape(M, ld)[:, :P]
                b = host[o * ostride:(o + 1) * ostride].reshape(M, ld)
                assert np.array_equal(a, b[:, :P]), (P, extra, small, o)
                assert np.isnan(b[:, P:]).all()


def test_recycled_result_buffers_are_page_locked(monkeypatch):
    """hostpool: a reused result buffer is registered with zk_host_register,
    results written into it are bitwise the unpinned ones, and eviction /
    clear() unregister it."""
    import gc

    from paper_2409_19156_b200 import hostpool

    pool = hostpool.ResultPool(1 << 30)
    monkeypatch.setattr(hostpool, "POOL", pool)
    req = zb.BatchRequest(modes=zb.full_mode_set(60), grid=zb.linear_radial_grid(3001))
    first = zb.evaluate_batch(req)[0].values  # fresh buffer (pageable, bounce path)
    want = first.copy()
    del first
    gc.collect()
    t = zb.evaluate_batch(req)[0]  # recycled -> page-locked -> direct DMA path
    assert [v for v in pool.pinned.values() if v] == [t.values.ctypes.data]
    assert np.array_equal(t.values, want)
    again = zb.evaluate_batch(req)[0]  # a second buffer (t still alive): fresh
    assert np.array_equal(again.values, want)
    del t, again
    gc.collect()
    pool.clear()
    assert not pool.pinned


def test_device_calls_are_cuda_graph_capturable():
    """The device-resident C-ABI calls (radial, 2-D, series) can be captured into
    a CUDA graph on the caller's stream (no host synchronisation or allocation
    inside a warm call) and replay bitwise (tools/graph_capture_check.py times
    it at config-2 size)."""
    import torch
    modes = zb.full_mode_set(30)
    n = np.array([md.n for md in modes], np.int32)
    m = np.array([md.m for md in modes], np.int32)
    M, P = n.size, 5000
    ctx = zb._lib.context(0)
    plan = zb._lib.plan_for(ctx, n, m)
    rho = torch.from_numpy(np.random.default_rng(3).uniform(size=P)).cuda()
    th = torch.from_numpy(np.random.default_rng(4).uniform(-3, 3, size=P)).cuda()
    coef = torch.from_numpy(np.random.default_rng(5).standard_normal(M)).cuda()
    out = torch.empty(M * P, dtype=torch.float64, device="cuda")
    out2 = torch.empty(M * P, dtype=torch.float64, device="cuda")
    f = torch.empty(P, dtype=torch.float64, device="cuda")
    A = zb._lib.ZK_ASYNC

    def calls():
        zb._lib.check(zb._lib.lib.zk_radial_eval(ctx.handle, plan.handle, rho.data_ptr(), P, 2, 1,
                                                 out.data_ptr(), P, M * P, A), "radial")
        zb._lib.check(zb._lib.lib.zk_zernike_eval(ctx.handle, plan.handle, rho.data_ptr(),
                                                  th.data_ptr(), P, 0, 0, out2.data_ptr(), P, 0,
                                                  A), "2d")
        zb._lib.check(zb._lib.lib.zk_series_eval(ctx.handle, plan.handle, rho.data_ptr(),
                                                 th.data_ptr(), P, 0, coef.data_ptr(), 1, M,
                                                 f.data_ptr(), P, A), "series")

    out = torch.empty(3 * M * P, dtype=torch.float64, device="cuda")  # orders 0..2
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    try:
        with torch.cuda.stream(s):
            calls()
        torch.cuda.synchronize()
        eager = (out.clone(), out2.clone(), f.clone())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            calls()
        out.zero_(), out2.zero_(), f.zero_()
        g.replay()
        torch.cuda.synchronize()
        for a, b in zip(eager, (out, out2, f)):
            assert torch.equal(a, b)
    finally:
        ctx.set_stream(None)
