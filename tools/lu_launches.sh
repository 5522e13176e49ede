# per-kernel launch list of one LU (n = 4096, 128 pencils) for CIRR_PANEL_QB=0 and 16
for qb in 0 16; do
  CIRR_PANEL_QB=$qb ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/lu_launch_qb$qb.csv python tools/lu_bench.py 4096 128 1 32 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/lu_launch_qb$qb.csv > gpurun_out/lu_launch_qb$qb.txt
done
