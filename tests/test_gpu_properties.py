"""Property-based parity on the GPU (hypothesis), in the style of the
reference's own property tests (tests/test_evaluate.py:224-251,
tests/test_batch.py:170-192): arbitrary mode requests and arbitrary binary64
points against the binary128 oracle (== the exact oracle) and the reference
algorithm. Examples are derandomized (stable across runs); tools/prop_hunt.py
explores fresh random requests against the same bitwise claim."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import zk_oracle as orc

pytestmark = pytest.mark.gpu

zb = pytest.importorskip("paper_2409_19156_b200")

mode = st.integers(0, 60).flatmap(lambda n: st.integers(0, n).map(lambda q: (n, -n + 2 * q)))
points = st.lists(st.floats(0.0, 1.0, allow_nan=False), min_size=1, max_size=40)


@given(st.lists(mode, min_size=1, max_size=30), points, st.integers(0, 3))
@settings(max_examples=60, deadline=None, derandomize=True)
def test_batch_matches_exact_oracle_at_arbitrary_points(modes, pts, k):
    grid = np.array(pts)
    t, _ = zb.evaluate_batch(zb.BatchRequest(modes=zb.as_mode_set(modes), grid=grid,
                                             deriv_order=k))
    exact = orc.quad_table(modes, grid, k)
    scale = np.maximum(1.0, np.abs(exact).max(axis=0))
    err = np.abs(t.values - exact).max(axis=0) / scale
    assert (err <= 1e-12).all()
    # bitwise the reference algorithm (zk/batch.py + zk/evaluate.py) once its
    # numpy pow is replaced by the correctly rounded power the kernels use:
    # numpy's SIMD pow is up to 1 ulp off, which the derivative assembly's
    # cancellation amplifies to a few ulps either way (tools/prop_hunt.py)
    # (below ~1e-250 the double-double power loses its low word to underflow,
    # so only the absolute size is checked there)
    ref_cr = orc.radial_batch(modes, grid, k, power=orc.cr_power)
    tiny = np.abs(ref_cr) < 1e-250
    bad = np.argwhere(~tiny & (t.values != ref_cr))
    assert bad.size == 0, [(modes[c], repr(grid[p]), k, repr(t.values[p, c]), repr(ref_cr[p, c]))
                           for p, c in bad[:4]]
    assert (np.abs(t.values - ref_cr)[tiny] <= 1e-250).all()


@given(st.lists(mode, min_size=1, max_size=12), points, st.integers(0, 2))
@settings(max_examples=30, deadline=None, derandomize=True)
def test_strategies_and_single_mode_agree_bitwise(modes, pts, k):
    grid = np.array(pts)
    ms = zb.as_mode_set(modes)
    a, _ = zb.batch_cached(zb.BatchRequest(modes=ms, grid=grid, deriv_order=k))
    b, _ = zb.batch_independent(zb.BatchRequest(modes=ms, grid=grid, deriv_order=k,
                                                strategy="independent"))
    assert np.array_equal(a.values, b.values)
    for col, md in enumerate(ms[:4]):
        assert np.array_equal(a.values[:, col], zb.radial_jacobi(md.n, md.m_abs, grid, k))


@given(mode, st.floats(0.0, 1.0, allow_nan=False), st.floats(-7.0, 7.0))
@settings(max_examples=60, deadline=None, derandomize=True)
def test_zernike_eval_is_radial_times_angular(md, rho, theta):
    n, m = md
    radial = zb.radial_jacobi(n, abs(m), [rho])[0]
    got = zb.zernike_eval(zb.make_mode(n, m), [rho], [theta])[0]
    ang = np.cos(m * theta) if m >= 0 else np.sin(abs(m) * theta)
    assert got == pytest.approx(radial * ang, abs=1e-13)
