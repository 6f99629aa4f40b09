"""The reference CLI `bench` timing (zk/cli.py:133-140: one warm-up, median of
3 wall times) of evaluate_batch through the plugin, n = 10..100 step 10 at 100
and 1,000 points, repeated R times: how often is the curve not strictly
increasing (acceptance criterion 9), and by how much do neighbours differ?
Needs baseline/_ref (the unmodified reference). python tools/crit9_probe.py [R]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
import zernkit  # noqa: E402

from paper_2409_19156_b200.zernkit_plugin import install  # noqa: E402

install(zernkit)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def timed(fn, reps=3):
    fn()
    s = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        fn()
        s.append(time.perf_counter_ns() - t0)
    return statistics.median(s)


bad = 0
for r in range(R):
    for grid_size in (100, 1000):
        grid = zernkit.linear_radial_grid(grid_size)
        for strategy in ("cached", "independent"):
            walls = []
            for n in range(10, 101, 10):
                req = zernkit.BatchRequest(modes=zernkit.full_mode_set(n), grid=grid,
                                           strategy=strategy)
                zernkit.evaluate_batch(req)
                walls.append(timed(lambda: zernkit.evaluate_batch(req)) / 1e3)
            ok = all(a < b for a, b in zip(walls, walls[1:]))
            bad += not ok
            if r < 2 or not ok:
                print(f"run {r} grid {grid_size} {strategy}: {'ok ' if ok else 'BAD'} "
                      + " ".join(f"{w:.0f}" for w in walls), flush=True)
print(f"{bad} non-increasing curves of {R * 4}")
