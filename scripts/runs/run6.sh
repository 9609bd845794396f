mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
echo "== MINB=4"; timeout 300 python scripts/perf_probe.py 2 10000,100000 sign,verify,keygen 5 2>&1 | tail -8
echo "== MINB=5"; DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_b5.so timeout 300 python scripts/perf_probe.py 2 10000,100000 sign 5 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sign_persistent -c 1 -o gpurun_out/prof_sign_r1b -f python scripts/perf_probe.py 2 100000 sign 1 > gpurun_out/ncu_full3.log 2>&1; tail -2 gpurun_out/ncu_full3.log
