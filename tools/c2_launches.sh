# config 2: host profile + ncu launch list of one solve_multi_batch of the 256 GEPs
python tools/c2_host_prof.py > gpurun_out/c2_host_prof.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
    python tools/config2_bench.py 1 --no-seq > gpurun_out/c2_bench_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/c2_launches.csv > gpurun_out/c2_launches.txt
