for K in 32 118 110 64; do
  for BN in 64 0; do
    echo "K=$K BN=$BN"; CIRR_SOLVE_BN=$BN python tools/lu_bench.py 4096 128 2 $K 2>&1 | tail -2
  done
done > gpurun_out/solve_ab.log 2>&1
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 >> gpurun_out/solve_ab.log
