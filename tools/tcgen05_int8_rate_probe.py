"""Rate of an int8 x int8 -> int32 GEMM on tcgen05 (the CUTLASS CuTe-DSL
Blackwell persistent dense-GEMM example shipped in the image, run as a
library kernel) at the shapes an Ozaki-style fp64-emulated config-5 Gram
would use: one slice product = (1920 x 131072) x (131072 x 1920), int32
exact over 131,072 points. Sizing data for DESIGN.md §9 (not product code).
python tools/tcgen05_int8_rate_probe.py"""
import importlib.util
import os

import cutlass

EX = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/cutlass/examples/"
      "python/CuTeDSL/blackwell/dense_gemm_persistent.py")
spec = importlib.util.spec_from_file_location("dense_gemm_persistent", EX)
mod = importlib.util.module_from_spec(spec)
os.chdir(os.path.dirname(EX))
spec.loader.exec_module(mod)

M = N = 1920
K = 131072
for tiler, cluster, two in (((256, 128), (2, 1), True), ((256, 256), (2, 1), True),
                            ((128, 128), (1, 1), False)):
    us = mod.run((M, N, K, 1), cutlass.Int8, cutlass.Int32, cutlass.Int32, "k", "k", "n",
                 mma_tiler_mn=tiler, cluster_shape_mn=cluster, use_2cta_instrs=two,
                 use_tma_store=False, warmup_iterations=3, iterations=20, skip_ref_check=True,
                 benchmark=True)
    tops = 2.0 * M * N * K / (us * 1e-6) / 1e12
    print(f"int8 GEMM {M}x{N}x{K} tiler {tiler} cluster {cluster} 2cta {two}: "
          f"{us:.1f} us = {tops:.0f} TOPS", flush=True)
