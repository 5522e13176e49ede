# time the LU with each prebuilt libcirr_<variant>.so swapped in
cp paper_2511_01927_b200/libcirr.so /tmp/libcirr_default.so
for f in default paper_2511_01927_b200/libcirr_*.so; do
  if [ "$f" != default ]; then cp "$f" paper_2511_01927_b200/libcirr.so; fi
  echo "variant $f"
  timeout 300 python tools/lu_bench.py 4096 128 2 32 2>&1 | grep rep1
  timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k getrf 2>&1 | tail -1
  cp /tmp/libcirr_default.so paper_2511_01927_b200/libcirr.so
done
