"""Host-side mirror of the reference API (validation, ordering, counters):
everything that must behave like zernkit before any kernel runs. CPU only."""

from fractions import Fraction

import numpy as np
import pytest

import paper_2409_19156_b200 as zb
from paper_2409_19156_b200.batch import BatchRequest


def test_mode_validation_exception_types():
    assert zb.make_mode(0, 0) == zb.Mode(0, 0)
    assert zb.make_mode(3, -1).m_abs == 1
    with pytest.raises(zb.ParityViolation):
        zb.make_mode(3, 2)
    with pytest.raises(zb.BoundViolation):
        zb.make_mode(2, 3)
    with pytest.raises(zb.DegreeViolation):
        zb.make_mode(-1, 0)
    assert issubclass(zb.ModeError, ValueError)


def test_full_mode_set_order(golden):
    assert [(md.n, md.m) for md in zb.full_mode_set(2)] == [
        (0, 0), (1, -1), (1, 1), (2, -2), (2, 0), (2, 2)]
    assert len(zb.full_mode_set(10)) == 66
    got = np.array([(md.n, md.m) for md in zb.full_mode_set(200)], dtype=np.int32)
    assert np.array_equal(got, golden["idx_full200"])
    with pytest.raises(zb.DegreeViolation):
        zb.full_mode_set(-1)


def test_dedup_plan_matches_reference(golden):
    for r in range(6):
        modes = zb.as_mode_set([tuple(x) for x in golden[f"idx_req{r}"].tolist()])
        plan = zb.dedup_plan(modes)
        assert np.array_equal(np.array(plan.unique_keys, np.int32).reshape(-1, 2),
                              golden[f"idx_req{r}_keys"])
        assert list(plan.scatter) == golden[f"idx_req{r}_scatter"].tolist()


def test_counters_hand_counts_and_closed_form():
    # reference tests/test_batch.py:55-62,99-105
    plan6 = zb.dedup_plan(zb.full_mode_set(6))
    assert zb.cached_step_counter(plan6, 0).recursion_steps == 4
    assert zb.independent_step_counter(plan6, 0).recursion_steps == 5
    assert len(plan6.unique_keys) == 16
    for N in range(0, 41):
        plan = zb.dedup_plan(zb.full_mode_set(N))
        want = sum(max(0, (N - a) // 2 - 1) for a in range(N + 1))
        assert zb.cached_step_counter(plan, 0).recursion_steps == want


def test_request_validation():
    grid = zb.linear_radial_grid(5)
    with pytest.raises(ValueError):
        BatchRequest(modes=zb.full_mode_set(2), grid=grid, deriv_order=4)
    with pytest.raises(ValueError):
        BatchRequest(modes=zb.full_mode_set(2), grid=grid, strategy="gpu")
    with pytest.raises(zb.GridError):
        BatchRequest(modes=zb.full_mode_set(2), grid=[2.0])
    req = BatchRequest(modes=[(2, 0), (4, 2)], grid=[0.5])
    assert req.modes == (zb.Mode(2, 0), zb.Mode(4, 2))
    cached = BatchRequest(modes=zb.full_mode_set(2), grid=grid, strategy="cached")
    indep = BatchRequest(modes=zb.full_mode_set(2), grid=grid, strategy="independent")
    # strategy mismatch is rejected before any device work
    with pytest.raises(ValueError):
        zb.batch_cached(indep)
    with pytest.raises(ValueError):
        zb.batch_independent(cached)


def test_single_mode_validation_before_device():
    with pytest.raises(ValueError):
        zb.radial_jacobi(2, 0, [0.5], 4)
    with pytest.raises(zb.ModeError):
        zb.radial_jacobi(3, 2, [0.5])
    with pytest.raises(zb.GridError):
        zb.radial_jacobi(2, 0, [1.5])
    with pytest.raises(ValueError):
        zb.radial_jacobi(2, -2, [0.5])
    with pytest.raises(ValueError):
        zb.zernike_eval(zb.make_mode(1, 1), [0.1, 0.2], [0.0])
    with pytest.raises(zb.GridError):
        zb.zernike_eval(zb.make_mode(1, 1), [0.1], [np.inf])
    with pytest.raises(ValueError):
        zb.jacobi_chain(-1, 0, 0, [0.0])
    with pytest.raises(ValueError):
        zb.jacobi_chain(2, -1, 0, [0.0])


def test_scalar_helpers():
    assert zb.jacobi_derivative_scale(5, 3, 1, 0) == 1.0
    assert zb.jacobi_derivative_scale(3, 2, 0, 1) == 3.0
    assert zb.jacobi_derivative_scale(2, 0, 0, 2) == 3.0
    assert zb.jacobi_derivative_scale(1, 4, 0, 2) == 0.0
    assert zb.jacobi_argument(np.array([0.0, 0.5, 1.0])).tolist() == [1.0, 0.5, -1.0]
    for n in range(0, 101):
        for m in range(-n, n + 1, 2):
            want = 0.0 if m else (1.0 if n % 4 == 0 else -1.0)
            assert zb.radial_at_zero(n, m) == want


def test_grids():
    g = zb.linear_radial_grid(100)
    assert np.array_equal(g, np.array([float(Fraction(i, 99)) for i in range(100)]))
    assert zb.rational_radial_grid(3) == (Fraction(0), Fraction(1, 2), Fraction(1))
    assert zb.radial_grid([]).size == 0
    with pytest.raises(zb.GridError):
        zb.radial_grid(np.zeros((2, 2)))
    with pytest.raises(zb.GridError):
        zb.linear_radial_grid(1)
    with pytest.raises(zb.GridError):
        zb.radial_grid([np.nan])


def test_empty_requests_need_no_device():
    # an empty grid or mode list is legal (zk/tables.py:22) and returns (0, M) / (P, 0)
    t, c = zb.evaluate_batch(BatchRequest(modes=zb.full_mode_set(3), grid=[]))
    assert t.values.shape == (0, 10)
    t, c = zb.evaluate_batch(BatchRequest(modes=(), grid=[0.1, 0.2]))
    assert t.values.shape == (2, 0) and c == zb.StepCounter(0, 0)


from hypothesis import given, settings, strategies as st  # noqa: E402

_mode = st.integers(0, 80).flatmap(lambda n: st.integers(0, n).map(lambda q: (n, -n + 2 * q)))


@given(st.lists(_mode, min_size=0, max_size=60), st.integers(0, 3))
@settings(max_examples=150, deadline=None, derandomize=True)
def test_native_plan_and_counters_on_arbitrary_requests(pairs, k):
    """Native planner == the reference algorithm (oracle port of zk/modes.py:
    108-125, zk/batch.py:69-94) on arbitrary requests, and the cached strategy
    never needs more recursion steps than the independent one (reference
    tests/test_batch.py: counter dominance)."""
    import zk_oracle as orc
    ms = zb.as_mode_set(pairs)
    plan = zb.dedup_plan(ms)
    keys, scatter = orc.unique_and_scatter([(md.n, md.m) for md in ms])
    assert list(plan.unique_keys) == [tuple(x) for x in keys]
    assert list(plan.scatter) == list(scatter)
    c = zb.cached_step_counter(plan, k)
    i = zb.independent_step_counter(plan, k)
    assert (c.recursion_steps, c.chain_count) == orc.step_counts(keys, k, True)
    assert (i.recursion_steps, i.chain_count) == orc.step_counts(keys, k, False)
    assert c.recursion_steps <= i.recursion_steps and c.chain_count <= i.chain_count
