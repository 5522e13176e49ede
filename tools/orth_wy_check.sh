python tools/orth_phases.py 4096 256 2 > gpurun_out/orth_wy.log 2>&1
python tools/orth_phases.py 8000 256 4 >> gpurun_out/orth_wy.log 2>&1
CIRR_ORTH_WY=0 python tools/orth_phases.py 4096 256 2 >> gpurun_out/orth_wy.log 2>&1
python -m pytest tests/test_gpu_kernels.py -q -x -k "orth" 2>&1 | tail -3 >> gpurun_out/orth_wy.log
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/orth_wy.log
