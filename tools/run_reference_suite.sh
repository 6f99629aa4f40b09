#!/usr/bin/env bash
# Run the reference's own test suite (zernkit tests/, unmodified) twice on a
# GPU box: stock (CPU numpy path) and with every hot-path name rebound to the
# B200 kernels (tools/ref_suite_plugin.py). Both outcomes are written under
# gpurun_out/ so the two pass/fail lists can be compared line by line.
#
# Prerequisites (build container, both git-ignored so they travel with gpurun):
#   cp -r /root/reference/pkg /tmp/refsrc
#   python -m pip install --no-index --no-build-isolation --no-deps \
#       --find-links /opt/wheelhouse --target baseline/_ref /tmp/refsrc
#   cp -r /root/reference/pkg/tests baseline/_ref/zernkit_tests
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T="$ROOT/baseline/_ref/zernkit_tests"
OUT="$ROOT/gpurun_out"
mkdir -p "$OUT"
[ -d "$T" ] || { echo "missing $T (see header)"; exit 2; }
cd "$T"
PYTHONPATH="$ROOT/baseline/_ref" python -m pytest -q -rf -p no:cacheprovider . \
  > "$OUT/ref_suite_stock.log" 2>&1
echo "stock rc=$?"
PYTHONPATH="$ROOT/tools:$ROOT/baseline/_ref" python -m pytest -q -rf -p no:cacheprovider \
  -p ref_suite_plugin . > "$OUT/ref_suite_b200.log" 2>&1
echo "b200 rc=$?"
tail -n 3 "$OUT/ref_suite_stock.log" "$OUT/ref_suite_b200.log"
