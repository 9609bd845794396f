set -e
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sign.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_api_and_scale.py -m gpu -x -q 2>&1 | tail -3
timeout 120 python scripts/perf_probe.py 2 10000,100000 sign 5 2>&1 | tail -3
timeout 120 python scripts/perf_probe.py 3,5 100000 sign 3 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sign_persistent -c 1 -o gpurun_out/prof_sign_r1c -f python scripts/perf_probe.py 2 100000 sign 1 > gpurun_out/ncu_full4.log 2>&1; tail -1 gpurun_out/ncu_full4.log
