set -e
mkdir -p gpurun_out
export DLB_NO_PEAK=1
timeout 600 ncu --set full --clock-control none -k regex:"k_" -c 80 -o /tmp/prof_kv -f python scripts/perf_probe.py 2 32768 keygen,verify 0 > gpurun_out/ncu_kv.log 2>&1 || (tail -5 gpurun_out/ncu_kv.log; exit 1)
python scripts/ncu_summary.py /tmp/prof_kv.ncu-rep gpurun_out/r01_kernels_keygen_verify > /dev/null
unset DLB_NO_PEAK
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err || (tail -5 gpurun_out/bench_r1e.err; exit 1)
timeout 300 python scripts/psi_sweep.py 2 1000000 0 2>&1 | tail -1
