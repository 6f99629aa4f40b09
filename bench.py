"""Benchmark of the hot path: fp64 Zernike radial basis evals/s.

Workload (BASELINE.json configs[1]), the same `config` object
for both arms: full mode set to n=100 (5,151 columns) x 1e5 radial points,
derivative order 0, the reference's linear grid i/(P-1). With N GPUs the 1e5
points are split into N contiguous shards (strong scaling, as config 2 states:
"1 B200 then sharded over 2/4/8"); no communication.

Arms
  default            libzk_b200 (CUDA, sm_100a) through the C ABI.
  --impl reference   the reference's own CPU path on the same config: the
                     unmodified zernkit.batch_cached(parallel=True) from
                     baseline/_ref (its ThreadPoolExecutor over alpha groups,
                     zk/batch.py:104-142) on the full 1e5-point grid every
                     step, plus one parallel=False (single-thread) call; the
                     bitwise-faithful numpy port (oracle/zk_oracle.py) only if
                     baseline/_ref is absent.

Secondary keys of the GPU line
  weak     1e5 points per GPU (N*1e5 global), the same kernel.
  c5fit    config 5's fit per step: series y = B c (K3) -> Gram [B y]^T[B y]
           (K4, DMMA) -> ONE allreduce of the packed triangle + B^T y (K5:
           the library's own NCCL communicator, zk_comm) -> Cholesky solve
           (K6), 1e6 disc points split over the N GPUs; per-phase device time.
  comm     the NCCL communicator's rank count.

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events on the launching stream, max over ranks. The 4.12 GB output is
32x the 126 MB L2, so no flush is needed between steps. `e2e` repeats the
metric through the same C ABI with host (pinned) buffers: every step copies
the grid H2D and lands the whole basis in host memory (the unique (n,|m|)
columns over PCIe, the repeated ones filled on the host) inside the timed
region.
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

# The image sets NCCL_DEBUG=VERSION, which makes every NCCL communicator init
# print its version banner to stdout -- the contract is ONE JSON line there.
# That level (only) is lowered to NONE before any communicator exists; an
# explicit WARN / INFO is left alone.
if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "NONE"
sys.path.insert(0, ROOT)

METRIC = "fp64 Zernike radial evals/s (points x modes)"
UNIT = "evals/s"
N_RES = 100
P_C2 = 100_000          # config 2: 1e5 radial points (split over the GPUs)
N_C5, P_C5 = 60, 1_000_000  # config 5: n<=60 2-D basis on 1e6 disc points
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


def c2_config() -> dict:
    """The workload both arms time -- identical objects, so the driver can
    compare the arms like for like."""
    return {"workload": f"config 2: full mode set n<={N_RES} (5151 modes) x {P_C2} radial points, "
                        "linear grid i/(P-1), k=0; N GPUs split the points into N contiguous "
                        "shards (strong scaling)",
            "global_points": P_C2, "modes": 5151, "deriv_order": 0,
            "grid": f"linear_radial_grid({P_C2})",
            "l2": "output 4.12 GB/step >> 126 MB L2 (no flush needed)"}


def host_info() -> dict:
    """The CPU the reference arm / cpu_baseline ran on."""
    info = {"cpu_count": os.cpu_count()}
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except Exception:
        info["affinity"] = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{"api": d.get("internal_api"), "threads": d.get("num_threads")}
                        for d in threadpool_info()]
    except Exception:
        info["blas"] = None
    info["reference_pool_workers"] = min(32, (os.cpu_count() or 1) + 4)  # ThreadPoolExecutor default
    return info


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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


def reference_call(points: int | None = None):
    """(run(parallel) -> None, P, M, kind): the reference's batch_cached on the
    config-2 request (zk/batch.py:104-142), or a bounded prefix of its grid
    when ``points`` is given (tests)."""
    zk = real_reference()
    if zk is not None:
        modes = zk.full_mode_set(N_RES)
        grid = zk.linear_radial_grid(P_C2)
        if points:
            grid = grid[:points]
        request = zk.BatchRequest(modes=modes, grid=grid)
        return (lambda par: zk.batch_cached(request, parallel=par)), grid.size, len(modes), \
            "reference"
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import zk_oracle as orc  # checker / CPU baseline only
    modes = orc.full_modes(N_RES)
    grid = orc.Workload(N_RES, P_C2).grid()
    if points:
        grid = grid[:points]
    return (lambda par: orc.radial_batch(modes, grid, 0, parallel=par)), grid.size, len(modes), \
        "port"


def ref_label(kind: str) -> str:
    if kind == "reference":
        return ("the unmodified reference, zernkit 0.1.0 batch_cached(parallel=True) "
                "from baseline/_ref")
    return "numpy port of zernkit.batch_cached(parallel=True) (oracle/zk_oracle.py)"


def timed_calls(run, warmup: int, reps: int) -> list[float]:
    out = []
    for i in range(warmup + reps):
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        if i >= warmup:
            out.append(dt)
    return out


def run_reference(args, world, rank):
    if rank != 0:
        return
    run, P, M, kind = reference_call(args.ref_points)
    times = timed_calls(lambda: run(True), args.warmup, max(1, args.steps))
    t = sum(times) / len(times)
    rate = P * M / t
    serial = None
    if not args.no_serial:  # the one-thread leg (parallel=False), one call
        ts = timed_calls(lambda: run(False), 0, 1)[0]
        serial = {"value": P * M / ts, "unit": UNIT, "ms_per_call": ts * 1e3, "threads": 1,
                  "call": "batch_cached(parallel=False)"}
    cores = host_cores()
    sample = (f"every step is the whole config-2 request ({P} points x {M} modes), "
              f"{ref_label(kind)}, ThreadPoolExecutor default workers min(32, cpu+4); "
              f"mean over {len(times)} steps after {args.warmup} warm-up")
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": c2_config() if not args.ref_points else
        dict(c2_config(), global_points=P, workload=f"test prefix of config 2: {P} points"),
        "parallelism": "host threads (reference ThreadPoolExecutor over alpha groups)",
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample, "host": host_info(), "serial_1thread": serial,
                         "step_ms": [round(x * 1e3, 1) for x in times]},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def max_over_ranks(dist, x: float, local: int) -> float:
    import torch
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_steps(step, stream, steps: int, warmup: int, dist):
    """Device time of `steps` calls of step() on `stream` (CUDA events),
    after `warmup` untimed calls; barrier + synchronize on both sides."""
    import torch
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(steps):
            step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    return ev0.elapsed_time(ev1)


def run_c5fit(args, world, rank, local, dist, stream, comm):
    """Config 5's fit, one step = series y = B c (K3) -> normal equations of
    [B y] (K4) -> K5 allreduce of the packed triangle + B^T y -> Cholesky
    (K6), on this rank's contiguous shard of 1e6 disc points."""
    import torch

    import paper_2409_19156_b200 as zb
    from paper_2409_19156_b200 import series as zs
    modes = zb.full_mode_set(N_C5)
    M = len(modes)
    rng = np.random.default_rng(0)
    rho_h = np.sqrt(rng.uniform(size=P_C5))
    th_h = 2 * np.pi * rng.uniform(size=P_C5)
    coef_h = rng.standard_normal(M)
    lo, hi = zb.shard_range(P_C5, world, rank)
    dev = torch.device("cuda", local)
    rho = torch.from_numpy(rho_h[lo:hi]).to(dev)
    th = torch.from_numpy(th_h[lo:hi]).to(dev)
    coef = torch.from_numpy(coef_h).to(dev)
    G = torch.zeros((M, M), dtype=torch.float64, device=dev)
    r = torch.zeros(M, dtype=torch.float64, device=dev)
    y = torch.empty(hi - lo, dtype=torch.float64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    # K3 through the C ABI on preallocated buffers (the phase is device time,
    # not the Python wrapper's argument handling)
    n_arr, m_arr = zb.modes.mode_arrays(modes)
    sctx = zb._lib.context(local)
    splan = zb._lib.plan_for(sctx, n_arr, m_arr)

    def series_k3():
        sctx.set_stream(stream.cuda_stream)
        zb._lib.check(zb._lib.lib.zk_series_eval(
            sctx.handle, splan.handle, rho.data_ptr(), th.data_ptr(), hi - lo, 0,
            coef.data_ptr(), 1, M, y.data_ptr(), hi - lo, zb._lib.ZK_ASYNC), "zk_series_eval")
    phase = np.zeros(4)
    x = None

    def step(record: bool):
        nonlocal x
        if record:
            ev[0].record(stream)
        series_k3()                                                  # K3
        if record:
            ev[1].record(stream)
        G.zero_()
        r.zero_()
        zs.gram_device(modes, rho, th, y, G, r)                      # K4
        if record:
            ev[2].record(stream)
        if comm is not None:                                         # K5
            zs.allreduce_normal_equations(G, r, comm=comm)
            Gs, rs = G, r
        else:
            Gs, rs = zs.allreduce_normal_equations(G, r)
        if record:
            ev[3].record(stream)
        x = zs.solve_normal(Gs, rs)                                  # K6
        if record:
            ev[4].record(stream)

    steps = max(1, min(args.fit_steps, args.steps))
    with torch.cuda.stream(stream):
        step(False)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        for _ in range(steps):
            step(True)
            torch.cuda.synchronize()
            phase += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    phase /= steps
    if dist:
        phase = np.array([max_over_ranks(dist, float(v), local) for v in phase])
    # the opt-in fp64-emulated Gram (gram_emulated.py: int8 slices x tcgen05 int8
    # GEMMs) on the same shard, timed the same way, with its deviation from K4
    emul = None
    try:
        from paper_2409_19156_b200.gram_emulated import gram_emulated_nm
        n5, m5 = zb.modes.mode_arrays(modes)
        with torch.cuda.stream(stream):
            Ge, _ = gram_emulated_nm(n5, m5, rho, th, y)  # JIT-compiles the GEMM once
            torch.cuda.synchronize()
            ev[0].record(stream)
            for _ in range(steps):
                Ge, be = gram_emulated_nm(n5, m5, rho, th, y)
            ev[1].record(stream)
            torch.cuda.synchronize()
        te = ev[0].elapsed_time(ev[1]) / steps
        if dist:
            te = max_over_ranks(dist, te, local)
        G.zero_()
        r.zero_()
        zs.gram_device(modes, rho, th, y, G, r)
        dev_g = float((Ge - G).abs().max() / G.diagonal().abs().max())
        emul = {"gram_ms": te, "max_abs_dev_vs_K4_over_max_diag": dev_g,
                "impl": "int8 slices (zk_emul_slices) x tcgen05 int8 GEMMs (CuTe-DSL library "
                        "kernel) -> fp64 recombination (zk_emul_accumulate); opt-in "
                        "ZK_GRAM_EMULATED=1"}
    except Exception as exc:  # noqa: BLE001 -- reported, the K4 numbers stand
        emul = {"unavailable": str(exc)[:200]}
    err = float((x.cpu() - torch.from_numpy(coef_h)).abs().max())
    nb = (M + 1 + 63) // 64  # 64 x 64 upper-triangle blocks of [B y] (zk_gram.cu BM)
    alg = 1.0 * P_C5 / world * (M + 1) * (M + 2)  # triangle of [B y]^T [B y], this rank
    return {"workload": f"config 5: 2-D basis n<={N_C5} ({M} modes) on {P_C5} disc points "
                        f"(rho=sqrt(U), theta=2 pi V, seed 0), {hi - lo} per GPU; y = B c, "
                        "c ~ N(0,1)",
            "steps": steps,
            "ms_per_step": float(phase.sum()),
            "phases_ms": {"series_K3": phase[0], "gram_K4": phase[1],
                          "allreduce_K5": phase[2], "solve_K6": phase[3]},
            "allreduce_bytes": 8 * int(zb._lib.lib.zk_gram_packed_count(M)),
            "allreduce_impl": ("libzk_b200 zk_gram_allreduce_comm (NCCL, packed triangle)"
                               if comm is not None else
                               "torch.distributed all_reduce of the packed triangle"),
            "gram_alg_tflops_per_gpu": alg / (phase[1] * 1e-3) / 1e12,
            "gram_executed_tiles": nb * (nb + 1) // 2,
            "fit_max_abs_err_vs_c": err,
            "gram_emulated": emul}


def run_gpu(args, world, rank, local):
    import torch

    import paper_2409_19156_b200 as zb
    from paper_2409_19156_b200 import _lib

    backend = os.environ.get("ZK_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # ZK_BENCH_BACKEND=gloo: functional check of the multi-rank path on one
        # GPU (NCCL refuses two ranks on one device); numbers from it are not
        # bench values
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    modes = zb.full_mode_set(N_RES)
    n_arr, m_arr = zb.modes.mode_arrays(modes)
    M = len(modes)
    ctx = _lib.context(local)
    plan = _lib.plan_for(ctx, n_arr, m_arr)
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream.cuda_stream)
    dev = f"cuda:{local}"

    # ---- headline: config 2, strong scaling (1e5 points over the N GPUs)
    grid = zb.linear_radial_grid(P_C2)
    lo, hi = zb.shard_range(P_C2, world, rank)
    P = hi - lo
    shard = np.ascontiguousarray(grid[lo:hi])
    d_rho = torch.from_numpy(shard).to(dev)
    out = torch.empty((M, P), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def step():
        _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, d_rho.data_ptr(), P, 0, 0,
                                           out.data_ptr(), P, 0, _lib.ZK_ASYNC), "zk_radial_eval")

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    launches0 = ctx.launches()
    t_ms = time_steps(step, stream, args.steps, args.warmup, dist)
    launches = ctx.launches() - launches0 - args.warmup
    clocks = sampler.stop() if sampler else None
    if dist:
        t_ms = max_over_ranks(dist, t_ms, local)
    ms_per_step = t_ms / args.steps
    value = P_C2 * M / (ms_per_step * 1e-3)  # every rank's points / max-over-ranks time

    # ---- roofline of the dominant (only) kernel: algorithmic bytes per launch
    alg_bytes = 8.0 * P * M + 8.0 * P  # basis writes + grid reads (this rank's launch)
    achieved = alg_bytes / (ms_per_step * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_traffic(f"radial_n{N_RES}_P{P}_k0")

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
        # every step timed on its own (each call synchronises): the median is the
        # headline -- the VM hosts show occasional slow host-memory phases --
        # with the mean and the extremes beside it
        samples = []
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            e2e_step()
            samples.append(time.perf_counter() - t0)
        te = float(np.median(samples))
        te_mean = float(np.mean(samples))
        if dist:
            te = max_over_ranks(dist, te, local)
            te_mean = max_over_ranks(dist, te_mean, local)
        host_view = np.ctypeslib.as_array(ctypes.cast(hbuf.value, ctypes.POINTER(ctypes.c_double)),
                                          shape=(M, P))
        e2e_ok = bool(np.array_equal(host_view, out.cpu().numpy()))  # every column
        del host_view
        _lib.lib.zk_host_free(hbuf)
        _lib.lib.zk_host_free(rbuf)
        U = plan.info()["U"]
        e2e = {"value": P_C2 * M / te, "unit": UNIT, "h2d_bytes_per_step": 8 * P,
               "d2h_bytes_per_step": 8 * P * U, "host_filled_bytes_per_step": 8 * P * (M - U),
               "ms_per_step": te * 1e3,
               "estimator": f"median of {e2e_steps} individually timed steps (each call "
                            f"synchronises); mean {te_mean * 1e3:.2f} ms, min "
                            f"{min(samples) * 1e3:.2f}, max {max(samples) * 1e3:.2f}",
               "path": "zk_radial_eval(ZK_HOST_INPUT|ZK_HOST_OUTPUT) into pinned host buffers: "
                       "chunked 2-stream pipeline, the U unique (n,|m|) columns cross PCIe, "
                       "the M-U repeated (+-m) columns are host copies of them (the "
                       "reference's unique->scatter, zk/batch.py:97-101)",
               "matches_device": e2e_ok}
    del out
    torch.cuda.empty_cache()

    # ---- weak scaling (secondary): 1e5 points per GPU
    weak = None
    if not args.no_weak:
        Pw = P_C2
        gw = zb.linear_radial_grid(P_C2 * world)
        d_w = torch.from_numpy(np.ascontiguousarray(gw[rank * Pw:(rank + 1) * Pw])).to(dev)
        out_w = torch.empty((M, Pw), dtype=torch.float64, device=dev)

        def wstep():
            _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, d_w.data_ptr(), Pw, 0, 0,
                                               out_w.data_ptr(), Pw, 0, _lib.ZK_ASYNC), "weak")

        tw = time_steps(wstep, stream, args.steps, args.warmup, dist)
        if dist:
            tw = max_over_ranks(dist, tw, local)
        weak = {"value": world * Pw * M / (tw / args.steps * 1e-3), "unit": UNIT,
                "ms_per_step": tw / args.steps, "points_per_gpu": Pw,
                "global_points": world * Pw}
        del out_w
        torch.cuda.empty_cache()

    # ---- the collective: the library's own NCCL communicator (zk_comm) when
    # every rank has its own GPU; torch.distributed (gloo) in the one-GPU check
    comm, comm_info = None, {"backend": backend if world > 1 else "none", "world_size": world}
    if backend == "nccl":
        try:
            if world > 1:
                obj = [_lib.Comm.unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                uid = obj[0]
            else:
                uid = _lib.Comm.unique_id()
            comm = _lib.Comm(ctx, uid, world, rank)
            comm_info.update({"impl": "libzk_b200 zk_comm (NCCL, dlopen libnccl.so.2)",
                              "nccl_version": _lib.nccl_version(),
                              "nccl_comm_nranks": comm.info()[0]})
        except Exception as exc:  # report, fall back to torch.distributed
            comm = None
            comm_info["zk_comm_error"] = str(exc)[:200]
    if dist is not None:
        comm_info["torch_pg_nranks"] = dist.get_world_size()
        if backend == "nccl":
            comm_info["torch_nccl_version"] = ".".join(map(str, torch.cuda.nccl.version()))

    fit = None
    if not args.no_fit:
        fit = run_c5fit(args, world, rank, local, dist, stream, comm)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu:
        run, Pc, Mc, kind = reference_call(args.ref_points)
        times = timed_calls(lambda: run(True), 1, 3)
        tc = statistics.median(times)
        cpu = {"value": Pc * Mc / tc, "unit": UNIT, "cores": host_cores(), "kind": kind,
               "sample": f"the whole config-2 request ({Pc} points x {Mc} modes), median of 3 "
                         f"after 1 warm-up (the reference's _timed_ns protocol, "
                         f"zk/cli.py:133-140); {ref_label(kind)}",
               "host": host_info()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": c2_config(),
        "parallelism": f"point shards x{world} ({P} points on rank 0), no communication",
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
        "weak": weak,
        "c5fit": fit,
        "comm": comm_info,
        "oracle_spot_check_max_abs": check,
    }
    print(json.dumps(line), flush=True)
    del comm
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-points", type=int, default=0,
                    help="tests only: time the reference on a prefix of the grid")
    ap.add_argument("--fit-steps", type=int, default=3, help="timed c5fit steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--no-fit", action="store_true")
    ap.add_argument("--no-serial", action="store_true", help="reference arm: skip the 1-thread call")
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
