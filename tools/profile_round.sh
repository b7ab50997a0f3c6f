#!/bin/bash
# Round profile on a GPU box: bench line, ncu launch list of one bench step, ncu --set full capture
# of the first Omega-sketch launch.  Usage (inside gpurun): bash tools/profile_round.sh r01
R=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$R.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_$R.log > gpurun_out/bench_$R.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$R.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ttm_s_tc_kernel -c 1 -o gpurun_out/full_$R \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$R.log 2>&1; echo "ncu full rc=$?"
