"""Benchmark of the hot path: fp64 Zernike radial basis evals/s.

Workload (BASELINE.json configs[1]): full mode set to n=100
(5,151 columns) x 1e5 radial points per GPU, derivative order 0, the
reference's linear grid i/(P-1); with N GPUs the global grid has N*1e5 points
and rank r evaluates its contiguous shard (weak scaling, no communication).

Arms
  default            libzk_b200 (CUDA, sm_100a) through the C ABI.
  --impl reference   the reference's own CPU path, zernkit.batch_cached with its
                     thread pool, on the host cores, bounded sample per step: the
                     unmodified package from baseline/_ref when it is installed
                     there, else its bitwise-faithful numpy port (oracle/zk_oracle.py).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events on the launching stream, max over ranks. The 4.12 GB output is
32x the 126 MB L2, so no flush is needed between steps. `e2e` repeats the
metric through the same C ABI with host (pinned) buffers: every step copies
the grid H2D and lands the whole 4.12 GB basis in host memory (the unique
(n,|m|) columns over PCIe, the repeated ones filled on the host) inside the
timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 Zernike radial evals/s (points x modes)"
UNIT = "evals/s"
N_RES = 100
P_PER_GPU = 100_000
STORE_CEILING_GBS = 6924.9  # tools/hbm_write_probe.cu, 32-B stores, 16 CTAs/SM


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(workload: str):
    """dram read+write bytes per launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
            except ValueError:
                continue
            for name, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def real_reference():
    """The unmodified reference package when it was installed into the
    git-ignored baseline/_ref (`pip install --target baseline/_ref`, DESIGN
    §7), else None (ZK_REF_ARM=port forces the numpy port)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.environ.get("ZK_REF_ARM", "auto") == "port" or not os.path.isdir(
            os.path.join(ref, "zernkit")):
        return None
    sys.path.insert(0, ref)
    try:
        import zernkit
    except Exception:
        return None
    finally:
        sys.path.remove(ref)
    return zernkit


def cpu_reference_rate(sample_points: int, reps: int, warmup: int = 1):
    """The reference's CPU path -- zernkit.batch_cached(parallel=True), its
    thread pool over alpha groups (zk/batch.py:104-142) -- on a bounded
    sample of the config-2 grid: the unmodified reference from baseline/_ref
    when present ("reference"), else the bitwise-faithful numpy port
    (oracle/zk_oracle.py, "port"). Returns (rate, s/step, points, modes, kind)."""
    zk = real_reference()
    if zk is not None:
        modes = zk.full_mode_set(N_RES)
        full = zk.linear_radial_grid(P_PER_GPU)
        pts = full[:: max(1, full.size // sample_points)][:sample_points]
        request = zk.BatchRequest(modes=modes, grid=pts)
        run, kind = (lambda: zk.batch_cached(request, parallel=True)), "reference"
    else:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import zk_oracle as orc  # checker / CPU baseline only
        modes = orc.full_modes(N_RES)
        full = orc.Workload(N_RES, P_PER_GPU).grid()
        pts = full[:: max(1, full.size // sample_points)][:sample_points]
        run, kind = (lambda: orc.radial_batch(modes, pts, 0, parallel=True)), "port"
    times = []
    for i in range(warmup + reps):
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    t = statistics.median(times)
    return pts.size * len(modes) / t, t, pts.size, len(modes), kind


def ref_label(kind: str) -> str:
    if kind == "reference":
        return ("the unmodified reference, zernkit 0.1.0 batch_cached(parallel=True) "
                "from baseline/_ref")
    return "numpy port of zernkit.batch_cached(parallel=True) (oracle/zk_oracle.py)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, world, rank):
    if rank != 0:
        return
    # bound the whole run to ~1-2 minutes (~0.3 s per 10^4-point step on 16
    # cores): the full --ref-sample per step up to 200 steps, fewer points
    # per step beyond that (small samples understate the CPU rate: numpy's
    # per-call overhead is amortised over fewer points)
    sample = int(min(args.ref_sample, max(1000, args.ref_sample * 200 // max(1, args.steps))))
    rate, t, npts, M, kind = cpu_reference_rate(sample, reps=max(1, args.steps),
                                                warmup=max(0, min(args.warmup, 1)))
    cores = host_cores()
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"full mode set n<={N_RES} ({M} modes) x {P_PER_GPU} radial points "
                               f"per GPU, k=0 (sampled: {npts} points per step)",
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{npts} of the {P_PER_GPU} config-2 grid points x {M} modes "
                                   f"per step; {ref_label(kind)}, "
                                   f"ThreadPoolExecutor default workers min(32, cpu+4)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def max_over_ranks(dist, x: float, local: int) -> float:
    import torch
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_gpu(args, world, rank, local):
    import torch

    import paper_2409_19156_b200 as zb
    from paper_2409_19156_b200 import _lib

    if os.environ.get("ZK_BENCH_BACKEND", "nccl") != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # ZK_BENCH_BACKEND=gloo: functional check of the multi-rank path on one
        # GPU (NCCL refuses two ranks on one device); numbers from it are not
        # bench values
        backend = os.environ.get("ZK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    modes = zb.full_mode_set(N_RES)
    n_arr, m_arr = zb.modes.mode_arrays(modes)
    M = len(modes)
    if args.scaling == "strong":  # config 2 as stated: 1e5 points split over the ranks
        Pg = P_PER_GPU
        lo, hi = zb.shard_range(Pg, world, rank)
    else:  # weak: 1e5 points per rank, the global grid grows with the world
        Pg = P_PER_GPU * world
        lo, hi = rank * P_PER_GPU, (rank + 1) * P_PER_GPU
    P = hi - lo
    grid_global = zb.linear_radial_grid(Pg)
    shard = np.ascontiguousarray(grid_global[lo:hi])

    ctx = _lib.context(local)
    plan = _lib.plan_for(ctx, n_arr, m_arr)
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream.cuda_stream)
    d_rho = torch.from_numpy(shard).to(f"cuda:{local}")
    out = torch.empty((M, P), dtype=torch.float64, device=f"cuda:{local}")
    torch.cuda.synchronize()

    def step():
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, d_rho.data_ptr(), P, 0, 0,
                                           out.data_ptr(), P, 0, _lib.ZK_ASYNC), "zk_radial_eval")

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    if dist:
        dist.barrier()
    t_ms = ev0.elapsed_time(ev1)
    clocks = sampler.stop() if sampler else None
    if dist:
        t_ms = max_over_ranks(dist, t_ms, local)
    ms_per_step = t_ms / args.steps
    value = Pg * M / (ms_per_step * 1e-3)  # every rank's points / max-over-ranks time

    # ---- roofline of the dominant (only) kernel: algorithmic bytes per launch
    alg_bytes = 8.0 * P * M + 8.0 * P  # basis writes + grid reads
    achieved = alg_bytes / (ms_per_step * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    workload = f"radial_n{N_RES}_P{P}_k0"
    traffic = load_traffic(workload)

    # sanity: the timed output is the real basis (spot check vs oracle)
    check = None
    if rank == 0 and not args.no_check:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import zk_oracle as orc
        idx = np.array([0, 1, P // 2, P - 1])
        ref = orc.radial_batch([(md.n, md.m) for md in modes], shard[idx], 0)
        got = out[:, torch.from_numpy(idx).to(out.device)].T.cpu().numpy()
        check = float(np.abs(got - ref).max())
        assert check <= 1e-11, f"bench output does not match the oracle: {check}"

    # ---- e2e: C ABI with pinned host buffers (H2D grid + D2H basis per step)
    e2e = None
    if not args.no_e2e:
        import ctypes
        hbuf = ctypes.c_void_p()
        _lib.check(_lib.lib.zk_host_alloc(8 * P * M, ctypes.byref(hbuf)), "zk_host_alloc")
        rbuf = ctypes.c_void_p()
        _lib.check(_lib.lib.zk_host_alloc(8 * P, ctypes.byref(rbuf)), "zk_host_alloc")
        ctypes.memmove(rbuf.value, shard.ctypes.data, 8 * P)
        flags = _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT

        def e2e_step():
            _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, rbuf.value, P, 0, 0,
                                               hbuf.value, P, 0, flags), "zk_radial_eval(host)")

        e2e_steps = max(3, min(args.steps, 10))
        e2e_step()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        te = (time.perf_counter() - t0) / e2e_steps
        if dist:
            te = max_over_ranks(dist, te, local)
        host_view = np.ctypeslib.as_array(ctypes.cast(hbuf.value, ctypes.POINTER(ctypes.c_double)),
                                          shape=(M, P))
        e2e_ok = bool(np.array_equal(host_view, out.cpu().numpy()))  # every column
        del host_view
        _lib.lib.zk_host_free(hbuf)
        _lib.lib.zk_host_free(rbuf)
        U = plan.info()["U"]
        e2e = {"value": Pg * M / te, "unit": UNIT, "h2d_bytes_per_step": 8 * P,
               "d2h_bytes_per_step": 8 * P * U, "host_filled_bytes_per_step": 8 * P * (M - U),
               "ms_per_step": te * 1e3,
               "path": "zk_radial_eval(ZK_HOST_INPUT|ZK_HOST_OUTPUT) into pinned host buffers: "
                       "chunked 2-stream pipeline, the U unique (n,|m|) columns cross PCIe, "
                       "the M-U repeated (+-m) columns are host copies of them (the "
                       "reference's unique->scatter, zk/batch.py:97-101)",
               "matches_device": e2e_ok}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu:
        rate, t, npts, _, kind = cpu_reference_rate(args.ref_sample, reps=3)
        cpu = {"value": rate, "unit": UNIT, "cores": host_cores(), "kind": kind,
               "sample": f"{npts} of {P} config-2 points x {M} modes, median of 3 after 1 warm-up; "
                         f"{ref_label(kind)}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"full mode set n<={N_RES} ({M} modes) x {P} radial points per GPU "
                               f"(linear grid i/(P-1), global {Pg} points sharded), k=0",
                   "global_points": Pg, "modes": M, "deriv_order": 0,
                   "parallelism": f"point shards x{world}, no communication",
                   "l2": "output 4.12 GB/step >> 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy r+w)",
                     "alg_bytes_per_launch": alg_bytes,
                     # the output is write-only: the copy peak (r+w) understates a
                     # pure-store kernel's ceiling; best incompressible streaming-store
                     # kernel measured in round 1 (profiles/r01_hbm_write_probe.txt)
                     "store_ceiling_gbs": STORE_CEILING_GBS,
                     "frac_of_store_ceiling": achieved / STORE_CEILING_GBS},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "oracle_spot_check_max_abs": check,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample", type=int, default=10_000,
                    help="points per reference step (bounded CPU sample)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: 1e5 points per GPU (default); strong: 1e5 points in total")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_gpu(args, world, rank, local)


if __name__ == "__main__":
    main()
