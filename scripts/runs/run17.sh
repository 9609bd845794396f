set -e
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_sign.py tests/test_gpu_edges.py tests/test_gpu_api_and_scale.py -m gpu -x -q 2>&1 | tail -2
echo "== MINB=5 (default)"; DLB_NO_PEAK=1 timeout 200 python scripts/perf_probe.py 2 10000,100000,400000 sign 5 2>&1 | tail -3
echo "== MINB=4"; DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_mb4.so DLB_NO_PEAK=1 timeout 200 python scripts/perf_probe.py 2 10000,100000,400000 sign 5 2>&1 | tail -3
echo "== L3/L5"; DLB_NO_PEAK=1 timeout 200 python scripts/perf_probe.py 3,5 100000 sign 5 2>&1 | tail -2
