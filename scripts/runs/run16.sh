set -e
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_sign.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -2
DLB_NO_PEAK=1 timeout 200 python scripts/perf_probe.py 2 1000,10000,30000,100000 sign 5 2>&1 | tail -4
timeout 200 python scripts/psi_sweep.py 2 10000 0,10240,20480,30720,40960,61440 2>&1 | tail -6
DLB_NO_PEAK=1 timeout 200 python scripts/perf_probe.py 3,5 10000 sign 5 2>&1 | tail -2
