#!/bin/bash
# Final-state ncu captures of every kernel family (run on the GPU box from the
# repo root; each program is run once plain first, as the profiling recipe asks).
set -u
out=gpurun_out/prof
mkdir -p $out
ONLY=${ONLY:-}
run() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  if [ -n "$ONLY" ] && ! echo "$name" | grep -qE "$ONLY"; then return; fi
  "$@" > $out/$name.plain.log 2>&1 || { echo "$name: plain run failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $out/$name "$@" \
      > $out/$name.ncu.log 2>&1
  echo "$name: ncu rc=$?"
  # keep the evidence small enough to travel back: raw metrics as CSV + a SASS
  # execution profile; drop the full report
  ncu -i $out/$name.ncu-rep --page raw --csv > $out/$name.raw.csv 2>/dev/null
  ncu -i $out/$name.ncu-rep --page source --csv --print-source sass > $out/$name.sass.csv 2>/dev/null
  gzip -f $out/$name.sass.csv
  rm -f $out/$name.ncu-rep
}
run k1_c2      radial_basis  2 python tools/run_config.py 100 100000 0 0 3
run k1_c3_k2   radial_basis  2 python tools/run_config.py 100 100000 2 0 3
run k1_c3_k3   radial_basis  2 python tools/run_config.py 100 100000 3 0 3
run k1_c3_all  radial_basis  2 python tools/run_config.py 100 100000 3 1 3
run k1_c4      radial_basis  2 python tools/run_config.py 200 10000 0 0 3
run k2_c5      radial_basis  2 python tools/run_config.py 60 1000000 0 0 3 1
run k3_series  "series_(k0_)?kernel" 2 python tools/run_series.py
run k4_syrk    "syrk_(tma|partial)"  0 python tools/run_gram.py
run k4_reduce  syrk_reduce   0 python tools/run_gram.py
run k3_series_dmma series_dmma  2 python tools/run_misc.py dmma
run x_chain    jacobi_chain  2 python tools/run_misc.py chain
run x_direct   direct_kernel 2 python tools/run_misc.py direct
run x_ztt      ztt_kernel    2 python tools/run_misc.py ztt
run x_dd       radial_dd     2 python tools/run_misc.py dd
