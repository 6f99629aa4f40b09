"""Cold-start cost of the numpy-level API in a fresh process: package import
(ctypes load of libzk_b200.so), CUDA context creation, plan upload, first
launch, then a warm call -- the counterpart of ZERNIPAX's ~400 ms first-call
JIT."""
import os
import sys
import time

t0 = time.perf_counter()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19156_b200 as zb  # noqa: E402
from paper_2409_19156_b200 import _lib  # noqa: E402

t1 = time.perf_counter()
ctx = _lib.context()
t2 = time.perf_counter()
modes = zb.full_mode_set(20)
n, m = zb.modes.mode_arrays(modes)
_lib.plan_for(ctx, n, m)
t3 = time.perf_counter()
req = zb.BatchRequest(modes=modes, grid=zb.linear_radial_grid(1000))
zb.evaluate_batch(req)
t4 = time.perf_counter()
zb.evaluate_batch(req)
t5 = time.perf_counter()
print(f"import {1e3*(t1-t0):.0f} ms | context {1e3*(t2-t1):.0f} ms | plan {1e3*(t3-t2):.1f} ms | "
      f"first C1 call {1e3*(t4-t3):.1f} ms | warm C1 call {1e3*(t5-t4):.2f} ms | "
      f"torch imported: {'torch' in sys.modules}")
