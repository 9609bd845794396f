cd /root/repo
export DLB_NO_PEAK=1
timeout 900 python -m pytest tests/test_gpu_sign.py tests/test_gpu_edges.py tests/test_gpu_api_and_scale.py -m gpu -x -q 2>&1 | tail -2
LEVELS=2,3,5 SIZES=10000,100000 VARIANTS=prev bash scripts/runs/ab.sh
SIZES=1000,1000000 VARIANTS=prev bash scripts/runs/ab.sh
timeout 300 python scripts/latency_probe.py 2>&1 | grep -E "n=    1 |n=   10|n=  100|n= 1000" | cut -c1-32
