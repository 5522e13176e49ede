#!/bin/bash
CMD="python tools/lu_bench.py 4096 128 1 32"
$CMD > gpurun_out/lu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_launches2.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:panel2_kernel -s 5 -c 1 -o gpurun_out/prof_panel $CMD > gpurun_out/ncu_panel.log 2>&1
echo rc=$?
