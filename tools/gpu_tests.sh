set -x
nvidia-smi --query-gpu=name,memory.used --format=csv
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_kats.py -q -m gpu 2>&1 | tail -30
