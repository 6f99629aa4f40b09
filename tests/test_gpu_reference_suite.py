"""The reference's OWN test suite, run with its five hot-path names rebound to
the B200 path (tools/ref_suite_plugin.py -> zernkit_plugin.install).

Needs the unmodified reference installed in the git-ignored baseline/_ref
with its tests/ copied to baseline/_ref/zernkit_tests (recipe in
tools/run_reference_suite.sh); skipped when that is absent. The only allowed
failures are the two acceptance criteria that fail by design on the stock
CPU path too (profiles/r01_reference_suite/stock_cpu.log)."""

import os
import re
import subprocess
import sys
import time

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "zernkit_tests")
FAIL_BY_DESIGN = {
    "test_acceptance.py::test_criterion_7_strict_step_dominance",
    "test_acceptance.py::test_criterion_8_zero_deviation_at_153_bits",
}
TIMING_FLAKY = "test_acceptance.py::test_criterion_9_bench_shape"


@pytest.mark.skipif(not os.path.isdir(TESTS), reason="reference suite not installed in baseline/_ref")
def test_reference_suite_on_the_b200_path():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tools"), REF]))
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-rf", "-p", "no:cacheprovider",
         "-p", "ref_suite_plugin", "."],
        cwd=TESTS, env=env, capture_output=True, text=True, timeout=900)
    out = proc.stdout + proc.stderr
    failed = set(re.findall(r"^FAILED (\S+)", out, re.M))
    # criterion 9 asserts that the CLI bench's wall time (median of 3) rises
    # strictly with n for calls of 40-150 us whose neighbours differ by ~5-7 us
    # at 100 points: timing-flaky on the stock CPU path as well (SURVEY.md fact
    # 1); tools/crit9_probe.py measured 6 of 80 such curves non-increasing on a
    # quiet box. A failure is re-run on its own (after a pause) up to four times
    # before it counts.
    rerun_passed = 0
    if TIMING_FLAKY in failed:
        for attempt in range(4):
            print(f"criterion 9 failed in the suite run; re-run {attempt + 1}")
            time.sleep(2.0)
            again = subprocess.run(
                [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                 "-p", "ref_suite_plugin", TIMING_FLAKY],
                cwd=TESTS, env=env, capture_output=True, text=True, timeout=300)
            if again.returncode == 0:
                failed.discard(TIMING_FLAKY)
                rerun_passed = 1
                break
    assert failed <= FAIL_BY_DESIGN, out[-4000:]
    m = re.search(r"B200 kernel launches during the reference suite: (\d+)", out)
    assert m and int(m.group(1)) > 1000, out[-2000:]  # the GPU path really ran
    passed = re.search(r"(\d+) passed", out)
    assert passed and int(passed.group(1)) + rerun_passed >= 157, out[-2000:]
