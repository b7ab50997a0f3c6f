for ab in 0 1 2; do
timeout 600 ncu --clock-control none -k regex:"sketch1_core0_kernel|ttm_s_h16_kernel" --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/fab_$ab.csv python tools/kbench_fused.py $ab > gpurun_out/fab_$ab.log 2>&1
done
