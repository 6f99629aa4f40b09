"""CLI on the GPU path: argument/validation errors (exit 2)
and I/O errors (exit 3) need no device; the evaluation/timing commands
are GPU tests with the reference's CSV/JSON schemas."""

import csv
import json

import numpy as np
import pytest
from click.testing import CliRunner

from paper_2409_19156_b200.cli import BENCH_HEADER, main


def _write(path, lines):
    path.write_text("\n".join(lines) + "\n")
    return str(path)


def test_usage_errors_exit_2(tmp_path):
    modes = _write(tmp_path / "m.txt", ["2 0", "3 2"])  # (3, 2) violates parity
    rho = _write(tmp_path / "r.txt", ["0.5"])
    res = CliRunner().invoke(main, ["eval", "--modes", modes, "--rho", rho])
    assert res.exit_code == 2 and "invalid mode" in res.output
    bad = _write(tmp_path / "b.txt", ["1 2 3"])
    res = CliRunner().invoke(main, ["eval", "--modes", bad, "--rho", rho])
    assert res.exit_code == 2
    res = CliRunner().invoke(main, ["bench", "--n-min", "5", "--n-max", "2"])
    assert res.exit_code == 2
    res = CliRunner().invoke(main, ["bench", "--method", "bogus"])
    assert res.exit_code == 2


def test_io_errors_exit_3(tmp_path):
    rho = _write(tmp_path / "r.txt", ["0.5"])
    res = CliRunner().invoke(main, ["eval", "--modes", str(tmp_path / "missing.txt"),
                                    "--rho", rho])
    assert res.exit_code == 3


@pytest.mark.gpu
def test_eval_csv_and_json_match_oracle(tmp_path):
    import zk_oracle as orc
    pairs = [(0, 0), (3, -1), (3, 1), (4, 2), (6, -4)]
    modes = _write(tmp_path / "m.txt", [f"{n} {m}" for n, m in pairs])
    pts = [0.0, 0.25, 0.5, 1.0]
    ths = [0.0, 1.0, -2.0, 3.0]
    rho = _write(tmp_path / "r.txt", [repr(x) for x in pts])
    th = _write(tmp_path / "t.txt", [repr(x) for x in ths])
    out = tmp_path / "o.csv"
    res = CliRunner().invoke(main, ["eval", "--modes", modes, "--rho", rho, "--k", "1",
                                    "--output", str(out)])
    assert res.exit_code == 0, res.output
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["rho"] + [f"R_{n}_{m}" for n, m in pairs]
    got = np.array([[float(v) for v in r[1:]] for r in rows[1:]])
    ref = orc.radial_batch(pairs, np.array(pts), 1)
    assert np.abs(got - ref).max() <= 1e-13 + 1e-12 * np.abs(ref).max()
    res = CliRunner().invoke(main, ["eval", "--modes", modes, "--rho", rho, "--theta", th,
                                    "--format", "json"])
    assert res.exit_code == 0, res.output
    payload = json.loads(res.output)
    assert payload["modes"] == [list(p) for p in pairs] and payload["deriv_order"] == 0
    ref2 = orc.basis_2d(pairs, np.array(pts), np.array(ths))
    assert np.abs(np.array(payload["values"]) - ref2).max() <= 1e-13


def test_accuracy_usage_errors():
    res = CliRunner().invoke(main, ["accuracy", "--n-max", "151"])  # zk/cli.py:40 guard
    assert res.exit_code == 2


@pytest.mark.gpu
def test_accuracy_matches_reference_study(golden, tmp_path):
    """The reference's own accuracy CSV (golden: zernkit run_accuracy(24, all
    methods, 100 points, k<=1) with the exact oracle) against ours (GPU
    methods, double-double reference): same rows; the errors are mostly
    identical and otherwise differ by an ulp of the evaluated value (rho**m
    rounding), far below the north_star tolerance."""
    out = tmp_path / "acc.csv"
    res = CliRunner().invoke(main, ["accuracy", "--n-max", "24", "--k-max", "1",
                                    "--output", str(out)])
    assert res.exit_code == 0, res.output
    rows = list(csv.reader(open(out)))
    assert tuple(rows[0]) == ("n", "m", "k", "method", "max_abs_err")
    meth = ("jacobi", "direct", "ztt")
    got = [(int(r[0]), int(r[1]), int(r[2]), meth.index(r[3])) for r in rows[1:]]
    assert np.array_equal(np.array(got, np.int32), golden["acc_rows"])
    err = np.array([float(r[4]) for r in rows[1:]])
    ref = golden["acc_err"]
    for mi in (0, 2):  # ztt seeds are rho**q: every pow rounding shows up there
        sel = golden["acc_rows"][:, 3] == mi
        assert np.mean(err[sel] == ref[sel]) > (0.9 if mi == 0 else 0.5), meth[mi]
        assert np.abs(err[sel] - ref[sel]).max() <= 1e-13, meth[mi]
    sel = golden["acc_rows"][:, 3] == 1  # direct sum: same Horner arithmetic; rho**low rounding
    assert np.abs(err[sel] - ref[sel]).max() <= 1e-13 + 0.05 * ref[sel].max()


@pytest.mark.gpu
def test_bench_records(tmp_path):
    out = tmp_path / "b.csv"
    res = CliRunner().invoke(main, ["bench", "--n-min", "10", "--n-max", "30", "--step", "10",
                                    "--grid-size", "100", "--reps", "3", "--output", str(out)])
    assert res.exit_code == 0, res.output
    rows = list(csv.reader(open(out)))
    assert tuple(rows[0]) == BENCH_HEADER
    assert len(rows) == 1 + 3 * 2
    by = {(r[1], int(r[2])): int(r[5]) for r in rows[1:]}
    res = CliRunner().invoke(main, ["bench", "--n-min", "30", "--n-max", "30", "--grid-size", "100",
                                    "--method", "jacobi", "--method", "direct", "--method", "ztt",
                                    "--reps", "3", "--output", str(out)])
    assert res.exit_code == 0, res.output
    assert {r[0] for r in list(csv.reader(open(out)))[1:]} == {"jacobi", "direct", "ztt"}
    for n in (10, 20, 30):
        assert by[("cached", n)] <= by[("independent", n)]
        assert by[("cached", n)] == sum(max(0, (n - a) // 2 - 1) for a in range(n + 1))


def test_precision_points_to_the_reference():
    res = CliRunner().invoke(main, ["precision", "--n-max", "10"])
    assert res.exit_code == 2 and "reference" in res.output
