set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_keygen_verify.py -m gpu -x -q 2>&1 | tail -30
