#!/bin/bash
# --set full of LU trailing-update launches of zgemm_sub_tma<64> (tools/lu_bench.py: n = 4096, 128 pencils)
CMD="python tools/lu_bench.py 4096 128 1 32"
$CMD > gpurun_out/r02_lu_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_lu_launches.csv \
    $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:zgemm_sub_tma -s 22 -c 2 \
    -o gpurun_out/r02_lu_gemm_full $CMD > gpurun_out/r02_lu_gemm_full.log 2>&1
echo rc=$?
