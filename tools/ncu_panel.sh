#!/bin/bash
# LU of 128 config-4 pencils (lu_bench.py), then one full ncu capture of a
# panel2_kernel launch early in the factorisation (tall panel) and one late.
CMD="python tools/lu_bench.py 4096 128 1 32"
$CMD > gpurun_out/lu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:panel2_kernel -s 2 -c 1 -o gpurun_out/prof_panel_early $CMD > gpurun_out/ncu_panel.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:panel2_kernel -s 40 -c 1 -o gpurun_out/prof_panel_mid $CMD >> gpurun_out/ncu_panel.log 2>&1
echo rc=$?
