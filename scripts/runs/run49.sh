cd /root/repo
export DLB_NO_PEAK=1
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_sign.py tests/test_gpu_keygen_verify.py tests/test_gpu_mldsa.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -2
LEVELS=2,3,5 SIZES=100000,1000000 VARIANTS="prev" bash scripts/runs/ab.sh
