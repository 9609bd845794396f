timeout 600 python -m pytest tests/test_gpu_sign.py tests/test_gpu_keygen_verify.py tests/test_gpu_primitives.py -m gpu -x -q 2>&1 | tail -3
echo "== WIDE"; timeout 300 python scripts/perf_probe.py 2 10000,100000 sign,verify,keygen 5 2>&1 | tail -6
echo "== HI"; DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_hi.so timeout 300 python scripts/perf_probe.py 2 10000,100000 sign,verify,keygen 5 2>&1 | tail -6
