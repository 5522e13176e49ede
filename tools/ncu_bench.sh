#!/bin/bash
# launch list of one bench step + one full capture of a k=512 LU trailing-update GEMM
# (each ncu pass only after the same command exited 0 without ncu)
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-variants"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 30000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:zgemm_sub_tma -s 8 -c 1 -o gpurun_out/prof_tma_gemm $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
