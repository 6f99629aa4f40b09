# Final-state evidence for profiles/: plain bench run, ncu launch list of the bench
# command (after it exited 0 without ncu), then one ncu --set full capture per kernel
# family (tools/profile_all.sh). Run on the GPU box from the repo root.
set -u
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_plain.log 2>&1 || { echo bench failed; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
bash tools/profile_all.sh
