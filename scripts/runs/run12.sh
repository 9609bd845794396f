set -e
mkdir -p gpurun_out
export DLB_NO_PEAK=1
timeout 600 ncu --set full --clock-control none -k regex:"k_" -c 60 -o /tmp/prof_kv -f python scripts/perf_probe.py 2 32768 keygen,verify 0 > gpurun_out/ncu_kv.log 2>&1 || (tail -5 gpurun_out/ncu_kv.log; exit 1)
python scripts/ncu_summary.py /tmp/prof_kv.ncu-rep gpurun_out/r01_kernels_keygen_verify > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sign|k_hash_mu" -c 4 -o gpurun_out/prof_sign_r1d -f python scripts/perf_probe.py 2 100000 sign 0 > gpurun_out/ncu_sign.log 2>&1 || (tail -5 gpurun_out/ncu_sign.log; exit 1)
python scripts/ncu_summary.py gpurun_out/prof_sign_r1d.ncu-rep gpurun_out/r01_kernels_sign > /dev/null
for lv in 3 5; do
timeout 600 ncu --set full --clock-control none -k regex:"k_sign_persistent" -c 1 -o /tmp/prof_sign_l$lv -f python scripts/perf_probe.py $lv 100000 sign 0 > gpurun_out/ncu_sign$lv.log 2>&1 || (tail -5 gpurun_out/ncu_sign$lv.log; exit 1)
python scripts/ncu_summary.py /tmp/prof_sign_l$lv.ncu-rep gpurun_out/r01_kernels_sign_l$lv > /dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_bench_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_under_ncu.json 2> gpurun_out/bench_under_ncu.err || (tail -5 gpurun_out/bench_under_ncu.err; exit 1)
du -sh gpurun_out; ls gpurun_out
