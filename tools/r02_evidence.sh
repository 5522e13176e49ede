#!/bin/bash
# One GPU call: full GPU suite, the bench line (both arms), smoke, then the ncu evidence.
TAG=${TAG:-_v4}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02${TAG}_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02${TAG}_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02${TAG}_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02${TAG}_bench.log
timeout 1200 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02${TAG}_bench_reference.log 2>&1
[ "${NCU:-1}" = 1 ] && TAG=$TAG timeout 2400 bash tools/ncu_r02.sh
echo done
