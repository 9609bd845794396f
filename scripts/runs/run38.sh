cd /root/repo
export DLB_NO_PEAK=1
timeout 900 python -m pytest tests/test_gpu_sign.py tests/test_gpu_edges.py tests/test_gpu_api_and_scale.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/psi_small.py 2 2>&1 | tail -6 | cut -c1-75
timeout 300 python scripts/latency_probe.py 2>&1 | tail -15
