#!/bin/bash
# ncu evidence for round 2 (run after the plain command exits 0):
#  1. launch list of one bench step (gpu__time_duration, serialised)
#  2. DRAM bytes of every kernel of one solve_multi (LU traffic summary)
#  3. --set full of one zgemm_sub_tma (DMMA), one ozaki_gemm_kernel (int8 trailing update) and one panel2_kernel
TAG=${TAG:-}
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-variants --no-per-config"
$CMD > gpurun_out/r02${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/r02${TAG}_launches.csv \
    $CMD > gpurun_out/r02${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/r02${TAG}_launches.csv > gpurun_out/r02${TAG}_launches_summary.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 900 --csv \
    --log-file gpurun_out/r02${TAG}_lu_traffic.csv $CMD > gpurun_out/r02${TAG}_ncu_traffic.log 2>&1
python tools/lu_traffic.py gpurun_out/r02${TAG}_lu_traffic.csv gpurun_out/r02${TAG}_lu_traffic.json > /dev/null
ncu --set full --clock-control none --import-source on -k regex:zgemm_sub_tma -s 300 -c 1 \
    -o gpurun_out/r02${TAG}_zgemm_full $CMD > gpurun_out/r02${TAG}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm_kernel -s 8 -c 1 \
    -o gpurun_out/r02${TAG}_ozaki_full $CMD >> gpurun_out/r02${TAG}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel2_kernel -s 20 -c 1 \
    -o gpurun_out/r02${TAG}_panel_full $CMD >> gpurun_out/r02${TAG}_ncu_full.log 2>&1
echo "rc=$?"
