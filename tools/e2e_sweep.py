"""e2e host-output sweep: zk_radial_eval(ZK_HOST_INPUT|ZK_HOST_OUTPUT) at config 2
into a page-locked (zk_host_alloc) and a pageable (pre-touched numpy) result,
over the staging-ring geometry (ZK_RING_SLOTS x ZK_RING_MB) and the old
land-in-place path (ZK_STAGED=0). Prints the median of 5 calls per setting."""
import ctypes
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

P, N = 100_000, 100
modes = zb.full_mode_set(N)
n, m = zb.modes.mode_arrays(modes)
M = len(modes)
ctx = _lib.context(0)
plan = _lib.plan_for(ctx, n, m)
grid = np.ascontiguousarray(zb.linear_radial_grid(P))
hbuf = ctypes.c_void_p()
_lib.check(_lib.lib.zk_host_alloc(8 * P * M, ctypes.byref(hbuf)), "alloc")
page = np.empty((M, P))
page.fill(0.0)
flags = _lib.ZK_HOST_INPUT | _lib.ZK_HOST_OUTPUT


def run(dst):
    _lib.check(_lib.lib.zk_radial_eval(ctx.handle, plan.handle, grid.ctypes.data, P, 0, 0, dst,
                                       P, 0, flags), "eval")


settings = [("staged=0", {"ZK_STAGED": "0"})]
for slots in (4, 6, 8, 12):
    for mb in (2, 4, 6, 8):
        settings.append((f"slots={slots} mb={mb}", {"ZK_STAGED": "1", "ZK_RING_SLOTS": str(slots),
                                                     "ZK_RING_MB": str(mb)}))
ref = None
for name, env in settings:
    os.environ.update(env)
    row = []
    for label, dst in (("pinned", hbuf.value), ("pageable", page.ctypes.data)):
        run(dst)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            run(dst)
            ts.append(time.perf_counter() - t0)
        row.append(f"{label} {statistics.median(ts) * 1e3:6.1f} ms (min {min(ts) * 1e3:5.1f})")
    host = np.ctypeslib.as_array(ctypes.cast(hbuf.value, ctypes.POINTER(ctypes.c_double)), shape=(M, P))
    if ref is None:
        ref = host.copy()
    ok = np.array_equal(host, ref) and np.array_equal(page, ref)
    print(f"{name:20s} " + " | ".join(row) + f" | bitwise {ok}", flush=True)
