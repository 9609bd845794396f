cd /root/repo
export DLB_NO_PEAK=1
DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_r0min.so timeout 900 python -m pytest tests/test_gpu_sign.py tests/test_gpu_edges.py tests/test_gpu_mldsa.py -m gpu -x -q 2>&1 | tail -2
LEVELS=2,3,5 SIZES=100000,1000000 VARIANTS="r0min" bash scripts/runs/ab.sh
