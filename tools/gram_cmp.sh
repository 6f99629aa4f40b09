#!/bin/bash
# usage: tools/gram_cmp.sh [P]: bitwise compare of the Gram (tools/gram_save.py) between
# the default TMA operand path and the cp.async ring (ZK_GRAM_TMA=0); P defaults to 2e5
P=${1:-200000}
mkdir -p gpurun_out
python tools/gram_save.py gpurun_out/ga.npy $P
ZK_GRAM_TMA=0 python tools/gram_save.py gpurun_out/gb.npy $P
python - <<PY
import numpy as np
a = np.load("gpurun_out/ga.npy"); b = np.load("gpurun_out/gb.npy"); M = 1891
G = (a - b)[:M * M].reshape(M, M)
bad = np.argwhere(np.abs(G) > 0)
print("P", $P, "bitwise", np.array_equal(a, b), "maxdiff", np.abs(a - b).max(), "nbad", len(bad),
      "blocks", sorted(set((int(i) // 64, int(j) // 64) for i, j in bad[:2000]))[:12])
PY
rm -f gpurun_out/ga.npy gpurun_out/gb.npy
