"""The CPU oracle (oracle/zk_oracle.py) pinned against golden vectors made by
the REAL reference (tests/golden/make_golden.py) and against the reference
tests' known-answer values. CPU only."""

import numpy as np
import pytest

import zk_oracle as orc


def _ulp_close(a, b, ulps=4):
    # bitwise on the generating host; a few ulp of slack elsewhere, because
    # numpy's SIMD pow differs across hosts
    scale = np.maximum(np.abs(b), np.finfo(np.float64).tiny)
    return bool((np.abs(a - b) <= ulps * np.spacing(scale)).all())


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_config1_full_set(golden, k):
    pts = golden["c1_grid_k0"] if k == 0 else golden["c1_grid_k123"]
    vals = orc.radial_batch(orc.full_modes(20), pts, k)[:, golden["c1_ucols"]]
    assert _ulp_close(vals, golden[f"c1_k{k}"])
    keys, _ = orc.unique_and_scatter(orc.full_modes(20))
    assert list(orc.step_counts(keys, k, True)) == golden[f"c1_k{k}_counter"].tolist()


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_config2_subsample(golden, k):
    pts = golden["c2_grid"] if k == 0 else golden["c2_grid"][::4]
    vals = orc.radial_batch(orc.full_modes(100), pts, k)[:, golden["c2_ucols"]]
    assert _ulp_close(vals, golden[f"c2_k{k}"])
    keys, _ = orc.unique_and_scatter(orc.full_modes(100))
    assert list(orc.step_counts(keys, k, True)) == golden[f"c2_k{k}_counter"].tolist()


def test_config4_high_order(golden):
    vals = orc.radial_batch(orc.full_modes(200), golden["c4_grid"], 0)[:, golden["c4_ucols"]]
    assert _ulp_close(vals, golden["c4_k0"])
    # the reference's own error against its exact oracle on these points
    assert np.abs(golden["c4_k0"] - golden["c4_exact"]).max() < 1.62e-13


def test_exact_oracle_restatement(golden):
    # restated bigint oracle == reference oracle_table on a slice of config 4
    ucols = golden["c4_ucols"]
    modes = orc.full_modes(200)
    keys = [modes[c] for c in ucols[::37]]
    pts = golden["c4_grid"][:6]
    got = orc.exact_table(keys, pts, 0)
    assert np.array_equal(got, golden["c4_exact"][:6, ::37])


def test_config5_basis_and_series(golden):
    modes = orc.full_modes(60)
    B = orc.basis_2d(modes, golden["c5_rho"], golden["c5_theta"])
    assert _ulp_close(B, golden["c5_B"])
    for k in (1, 2, 3):
        Bk = orc.basis_2d(modes, golden["c5_rho"], golden["c5_theta"], k)
        assert _ulp_close(Bk, golden[f"c5_B_k{k}"]), k
    f = B @ golden["c5_coef"]
    assert np.allclose(f, golden["c5_f"], rtol=1e-13, atol=1e-13)


def test_mode_indexing(golden):
    assert np.array_equal(np.array(orc.full_modes(200), dtype=np.int32), golden["idx_full200"])
    for r in range(6):
        req = [tuple(x) for x in golden[f"idx_req{r}"].tolist()]
        keys, scatter = orc.unique_and_scatter(req)
        assert np.array_equal(np.array(keys, np.int32).reshape(-1, 2), golden[f"idx_req{r}_keys"])
        assert scatter == golden[f"idx_req{r}_scatter"].tolist()
        for k in range(4):
            want = golden[f"idx_req{r}_counters"][k].tolist()
            assert list(orc.step_counts(keys, k, True)) + list(orc.step_counts(keys, k, False)) == want
        for k in (0, 2):
            got = orc.radial_batch(req, golden["idx_req_grid"], k)
            assert _ulp_close(got, golden[f"idx_req{r}_k{k}"])


def test_reference_known_answers():
    # tests/test_evaluate.py:28-40,60-64,104-111,264-266 of the reference
    assert np.all(orc.jacobi_chain(0, 3, 1, np.array([-1.0, 0.5]))[0] == 1.0)
    assert orc.jacobi_chain(1, 2, 0, np.array([-1.0]))[1][0] == -1.0
    assert orc.jacobi_chain(2, 0, 0, np.array([0.5]))[2][0] == -0.125
    assert orc.derivative_scale(3, 2, 0, 1) == 3.0
    assert orc.derivative_scale(2, 0, 0, 2) == 3.0
    assert orc.derivative_scale(1, 4, 0, 2) == 0.0
    g = np.linspace(0.0, 1.0, 7)
    for k in (1, 2, 3):
        assert np.all(orc.radial_single(0, 0, g, k) == 0.0)
    assert np.all(orc.radial_single(1, 1, g, 2) == 0.0)
    assert np.all(orc.radial_single(2, 2, g, 3) == 0.0)
    assert np.all(orc.radial_single(3, 3, g, 3) == 6.0)
    assert orc.jacobi_argument(np.array([0.0, 0.5, 1.0])).tolist() == [1.0, 0.5, -1.0]


def test_batch_equals_single_mode():
    # tests/test_batch.py:108-116 of the reference, on the oracle itself
    g = np.arange(37) / 36.0
    modes = orc.full_modes(10)
    table = orc.radial_batch(modes, g, 2)
    for col, (n, m) in enumerate(modes):
        assert np.array_equal(table[:, col], orc.radial_single(n, abs(m), g, 2))


def test_binary128_oracle_equals_exact_oracle(golden):
    # the fast binary128 oracle (oracle/zk_quad.c) reproduces the reference's
    # exact big-integer oracle bit for bit: all 16 x 10,201 golden n=200 values...
    modes = orc.full_modes(200)
    umodes = [modes[c] for c in golden["c4_ucols"]]
    assert np.array_equal(orc.quad_table(umodes, golden["c4_grid"], 0), golden["c4_exact"])
    # ...and every derivative order against the restated exact oracle
    pts = np.array([0.0, 1e-3, 0.1, 0.37, 0.5, 0.77, 0.93, 1.0])
    small = [(n, m) for n in range(0, 41) for m in range(-n, n + 1, 2)]
    for k in range(4):
        assert np.array_equal(orc.quad_table(small, pts, k), orc.exact_table(small, pts, k)), k


def test_cr_power_variant_differs_only_through_pow():
    """radial_batch(power=cr_power) -- the GPU's bitwise oracle -- equals the
    reference port wherever numpy's pow returned the correctly rounded power
    for every exponent the assembly uses, at every derivative order."""
    rng = np.random.default_rng(11)
    modes = [(n, m) for n in range(0, 31) for m in range(-n, n + 1, 2)]
    pts = rng.uniform(size=60)
    for k in range(4):
        a = orc.radial_batch(modes, pts, k)
        b = orc.radial_batch(modes, pts, k, power=orc.cr_power)
        for c, (n, m) in enumerate(modes):
            ma = abs(m)
            exps = range(max(ma - k, 0), ma + k + 1)
            same_pow = np.ones(pts.size, bool)
            for e in exps:
                same_pow &= orc.numpy_power(pts, e) == orc.cr_power(pts, e)
            assert np.array_equal(a[same_pow, c], b[same_pow, c]), (n, m, k)


def test_float_baselines_match_the_reference(golden):
    """The oracle's restatement of the reference's float baselines
    (zk/evaluate.py:189-247: direct Horner sum, Zernike three-term table) is
    bitwise the reference's output on the generating host."""
    pts = golden["base_pts"]
    modes = [tuple(int(x) for x in r) for r in golden["base_modes"]]
    for k in (0, 1, 2):
        got = np.stack([orc.direct_single(n, m, pts, k) for n, m in modes], axis=1)
        assert _ulp_close(got, golden[f"base_direct_k{k}"]), k
    assert _ulp_close(orc.ztt_table(modes, pts), golden["base_ztt"])


def test_jacobi_chain_matches_the_reference(golden):
    """oracle jacobi_chain == zk/evaluate.py:36-76 output, bitwise (pure
    +,-,*,/ in the reference's order: host independent)."""
    x = golden["chain_x"]
    for jm, al, be in golden["chain_cases"]:
        assert np.array_equal(orc.jacobi_chain(int(jm), int(al), int(be), x),
                              golden[f"chain_{jm}_{al}_{be}"]), (jm, al, be)
