"""GPU float baselines: the reference's direct sum and Zernike
three-term recursion, against the oracle restatements and the reference's
own baseline tests (tests/test_evaluate.py:133-180 of the reference)."""

import numpy as np
import pytest

import zk_oracle as orc

pytestmark = pytest.mark.gpu

zb = pytest.importorskip("paper_2409_19156_b200")


def test_direct_matches_reference_algorithm():
    grid = zb.linear_radial_grid(100)
    for k in range(4):
        for n, m in [(0, 0), (1, 1), (2, 0), (8, 2), (20, 4), (31, 7)]:
            got = zb.radial_direct(n, m, grid, k)
            ref = orc.direct_single(n, m, grid, k)
            scale = max(1.0, np.abs(ref).max())
            assert np.abs(got - ref).max() <= 1e-13 * scale, (n, m, k)
    assert zb.radial_direct(2, 0, [0.5])[0] == pytest.approx(-0.5, abs=1e-15)
    assert np.all(zb.radial_direct(0, 0, grid) == 1.0)
    assert np.all(zb.radial_direct(1, 1, grid, 2) == 0.0)  # zero polynomial


def test_direct_is_unstable_at_high_degree():
    # reference tests/test_evaluate.py:138-142: error > 1 at n = 80
    grid = zb.linear_radial_grid(100)
    exact = orc.quad_table([(80, 0)], grid, 0)[:, 0]
    assert np.abs(zb.radial_direct(80, 0, grid) - exact).max() > 1.0


def test_ztt_matches_reference_algorithm_and_oracle():
    grid = zb.linear_radial_grid(100)
    modes = [(n, m) for n in range(21) for m in range(n % 2, n + 1, 2)]
    got = zb.radial_ztt_table(zb.as_mode_set(modes), grid)
    ref = orc.ztt_table(modes, grid)
    assert np.abs(got - ref).max() <= 1e-14
    exact = orc.quad_table(modes, grid, 0)
    assert np.abs(got - exact).max() <= 1e-10  # reference tests/test_evaluate.py:157-161
    seeds = zb.linear_radial_grid(17)
    for q in (0, 1, 3, 7):
        assert np.allclose(zb.radial_ztt(q, q, seeds), seeds ** q, rtol=2e-16, atol=0)
    # signed and duplicated request columns, high degree
    req = zb.as_mode_set([(40, -2), (40, 2), (7, 3), (40, 2), (100, 0)])
    t = zb.radial_ztt_table(req, grid)
    assert np.array_equal(t[:, 0], t[:, 1]) and np.array_equal(t[:, 1], t[:, 3])
    r2 = orc.ztt_table([(40, 2), (7, 3), (100, 0)], grid)
    assert np.abs(t[:, [1, 2, 4]] - r2).max() <= 1e-12


def test_baseline_validation():
    with pytest.raises(zb.ModeError):
        zb.radial_direct(3, 2, [0.5])
    with pytest.raises(ValueError):
        zb.radial_ztt(2, -2, [0.5])
    with pytest.raises(zb.GridError):
        zb.radial_ztt_table(zb.full_mode_set(2), [1.5])


def test_double_double_reference_equals_exact_oracle(golden):
    """zk_radial_eval_dd (the GPU accuracy reference) reproduces the exact
    oracle: on the golden n=200 binary64 points, and -- every order -- at the
    exact rationals i/40 the reference's accuracy study uses."""
    from fractions import Fraction

    from paper_2409_19156_b200.accuracy import rational_grid_dd, reference_table
    modes = zb.full_mode_set(200)
    umodes = zb.as_mode_set([(modes[c].n, modes[c].m) for c in golden["c4_ucols"]])
    got = reference_table(umodes, golden["c4_grid"], None, 0)
    assert np.mean(got == golden["c4_exact"]) > 0.999
    assert np.abs(got - golden["c4_exact"]).max() <= 1e-15 * np.abs(golden["c4_exact"]).max()
    hi, lo = rational_grid_dd(41)
    small = [(n, m) for n in range(31) for m in range(n % 2, n + 1, 2)]
    pts = [Fraction(i, 40) for i in range(41)]
    for k in range(4):
        ref = reference_table(zb.as_mode_set(small), hi, lo, k)
        ex = orc.exact_table_rational(small, pts, k)
        assert np.mean(ref == ex) > 0.99, k
        assert np.abs(ref - ex).max() <= 1e-14 * max(1.0, np.abs(ex).max()), k


def test_baselines_match_reference_golden(golden):
    """GPU float baselines against outputs of the reference itself
    (tests/golden: radial_direct k <= 2, radial_ztt_table), within the
    baselines' own rounding (column-scaled 1e-13; the direct sum is unstable
    by design, so high-degree columns are compared relative to their size)."""
    pts = golden["base_pts"]
    modes = [tuple(int(x) for x in r) for r in golden["base_modes"]]
    for k in (0, 1, 2):
        ref = golden[f"base_direct_k{k}"]
        got = np.stack([zb.radial_direct(n, m, pts, k) for n, m in modes], axis=1)
        scale = np.maximum(1.0, np.abs(ref).max(axis=0))
        assert (np.abs(got - ref).max(axis=0) <= 1e-13 * scale).all(), k
    ref = golden["base_ztt"]
    got = zb.radial_ztt_table(zb.as_mode_set(modes), pts)
    assert np.abs(got - ref).max() <= 1e-14


def test_ztt_any_degree_global_level_table():
    """Beyond n = 256 the ZTT kernel keeps its level array in device memory
    (the reference's memoised recursion has no degree limit,
    zk/evaluate.py:211-241): same arithmetic, so columns shared with a
    register-table request (n <= 256) are bitwise equal, and n = 300..400
    match the oracle's restatement."""
    rng = np.random.default_rng(11)
    grid = np.concatenate([[0.0, 1.0], rng.uniform(size=200)])
    big = [(400, 0), (301, 1), (300, 300), (200, 4), (256, 2)]
    small = [(200, 4), (256, 2)]
    got = zb.radial_ztt_table(zb.as_mode_set(big), grid)
    reg = zb.radial_ztt_table(zb.as_mode_set(small), grid)
    assert np.array_equal(got[:, 3:], reg)
    ref = orc.ztt_table(big, grid)
    assert np.abs(got - ref).max() <= 1e-11
