"""bench.py's driver contract: one JSON line with the required keys, for the
reference arm (CPU, runs here) and the GPU arm (B200)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "cpu_baseline"}


def _run(args, timeout=600):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-points", "300"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    assert cb["host"]["cpu_count"] >= 1 and "affinity" in cb["host"] and "blas" in cb["host"]
    assert cb["serial_1thread"]["threads"] == 1 and cb["serial_1thread"]["value"] > 0
    assert len(cb["step_ms"]) == 2
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 == d["e2e"]["d2h_bytes_per_step"]
    assert d["scaling"] == "strong" and d["config"]["global_points"] == 300


def test_both_arms_share_the_config_object():
    """Without --ref-points the reference arm times the whole config-2 request
    and prints bench.c2_config() -- the very object the GPU arm prints."""
    sys.path.insert(0, ROOT)
    import bench
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"config": c2_config(),') == 1  # GPU arm
    assert 'c2_config() if not args.ref_points' in src  # reference arm
    c = bench.c2_config()
    assert c["global_points"] == 100_000 and c["modes"] == 5151 and c["deriv_order"] == 0
    run, P, M, kind = bench.reference_call()
    assert (P, M) == (100_000, 5151)


@pytest.mark.gpu
def test_gpu_arm_json_line():
    d = _run(["--steps", "5", "--warmup", "3", "--no-cpu"])
    assert BASE_KEYS <= set(d) and {"roofline", "gpu_launches", "clocks"} <= set(d)
    assert d["scaling"] == "strong" and d["config"]["global_points"] == 100_000
    assert d["weak"]["global_points"] == 100_000 and d["weak"]["value"] > 1e11
    f = d["c5fit"]
    assert set(f["phases_ms"]) == {"series_K3", "gram_K4", "allreduce_K5", "solve_K6"}
    assert f["fit_max_abs_err_vs_c"] < 1e-8
    assert f["allreduce_bytes"] == 8 * (1891 * 1892 // 2 + 1891)
    assert d["comm"]["nccl_comm_nranks"] == 1 and "libzk_b200" in f["allreduce_impl"]
    assert d["gpu_launches"] == 5 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.5 < r["frac"] < 1.3
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["matches_device"] is True and e["value"] > 1e9
    assert e["d2h_bytes_per_step"] + e["host_filled_bytes_per_step"] == 8 * 100_000 * 5151
    assert d["oracle_spot_check_max_abs"] <= 1e-11


def test_reference_arm_under_torchrun_prints_once():
    """N > 1 (driver launches the reference arm through torchrun too): rank 0
    alone runs and prints; the other ranks exit 0 without work."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "0", "--ref-points", "200"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


@pytest.mark.gpu
def test_gpu_arm_multi_rank_path_on_one_gpu():
    """The torchrun path of the GPU arm (barriers, max-over-ranks timing,
    rank-0 line) with two ranks sharing the one GPU through gloo -- a
    functional check of the code the driver's N-GPU runs take (NCCL itself
    needs one device per rank)."""
    env = dict(os.environ, ZK_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29563",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--no-e2e", "--fit-steps", "1"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["gpu_launches"] == 3
    assert d["config"]["global_points"] == 100_000  # strong: config 2's 1e5 points split
    assert d["roofline"]["alg_bytes_per_launch"] == 8.0 * 50_000 * 5151 + 8.0 * 50_000
    assert d["weak"]["global_points"] == 200_000  # weak: 1e5 per rank
    f = d["c5fit"]
    assert set(f["phases_ms"]) == {"series_K3", "gram_K4", "allreduce_K5", "solve_K6"}
    assert f["fit_max_abs_err_vs_c"] < 1e-8 and "torch.distributed" in f["allreduce_impl"]
    assert d["comm"]["torch_pg_nranks"] == 2
