#!/bin/bash
# full ncu capture of the LU trailing-update kernel (source-level stalls)
CMD="python tools/lu_bench.py 4096 128 1 32"
$CMD > gpurun_out/lu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:zgemm_sub -s 10 -c 1 -o gpurun_out/prof_lugemm2 $CMD > gpurun_out/ncu_lu.log 2>&1
echo rc=$?
