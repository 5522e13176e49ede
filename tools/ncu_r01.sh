#!/bin/bash
# ncu evidence for round 1: launch list of one bench step + a full capture of the trailing-update GEMM
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 1 -o gpurun_out/prof_gemm_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
