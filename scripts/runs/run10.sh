set -e
timeout 300 python -m pytest tests/test_gpu_sign.py tests/test_gpu_keygen_verify.py -m gpu -x -q 2>&1 | tail -2
timeout 200 python scripts/perf_probe.py 2 10000,100000 sign,verify,keygen 5 2>&1 | tail -6
timeout 200 python scripts/psi_sweep.py 2 10000 0,10240,15360,20480,30720,40960,75776 2>&1 | tail -7
timeout 200 python scripts/psi_sweep.py 2 100000,400000 0,75776 2>&1 | tail -4
