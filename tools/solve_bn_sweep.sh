# solve-pass time per tile width (CIRR_SOLVE_BN) with and without swizzled B boxes, n=4096 x 128 pencils
for SW in 0 1; do
  for K in 118 110 32; do
    for BN in 64 56 48 40 32; do
      echo "SW=$SW K=$K BN=$BN $(CIRR_SOLVE_BSWZ=$SW CIRR_SOLVE_BN=$BN python tools/lu_bench.py 4096 128 2 $K 2>&1 | tail -2 | head -1 | sed 's/.*solve/solve/')"
    done
  done
done
