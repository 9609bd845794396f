# quick GPU check: sign parity tests, throughput probe, dynamic instruction count of the sign kernel
cd /root/repo
export DLB_NO_PEAK=1
timeout 900 python -m pytest tests/test_gpu_sign.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/perf_probe.py ${LEVELS:-2} 10000,100000,1000000 sign 5 2>&1 | tail -${TAILN:-3}
timeout 300 ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_sign_persistent" -c 1 python scripts/perf_probe.py 2 100000 sign 0 2>&1 | grep -E "inst_executed|issue_active|single call"
