#!/bin/bash
# Per-pass ncu metrics of one cfg5 HOSVD step (DRAM throughput, tensor-pipe activity, duration) for
# the X-streaming kernels.  Usage (inside gpurun): bash tools/pass_table.sh r01
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --clock-control none -k regex:"ttm_s_tc_kernel|ttm_s_h16_kernel|ttm_t_tc_kernel|residual_tc_kernel|residual_h16_kernel|sketch1_core0_kernel|cs_" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  --csv --log-file gpurun_out/passes_$R.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_passes_$R.log 2>&1
echo "ncu passes rc=$?"
