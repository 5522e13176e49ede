# A/B of libcirr builds (CIRR_LIB) on the config-4 LU + one K=118 solve pass
for L in base none swz tst cur base cur; do
  if [ $L = cur ]; then unset CIRR_LIB; else export CIRR_LIB=$PWD/paper_2511_01927_b200/libcirr_$L.so; fi
  echo "$L: $(python tools/lu_bench.py 4096 128 3 118 2>&1 | tail -2 | head -1)"
done
