# LU step width (panels per multi-level step) at n = 4096, 128 pencils
for pb in 8 16 12; do
  echo "PB=$pb"; CIRR_LU_PB=$pb python tools/lu_bench.py 4096 128 2 32 2>&1 | tail -2
done > gpurun_out/lu_pb.log 2>&1
