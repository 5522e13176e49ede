#!/bin/bash
# bench line + ncu launch list of one bench step + full capture of the LU trailing-update kernel
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:zgemm_sub_tma -s 80 -c 1 -o gpurun_out/prof_tma_gemm $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
