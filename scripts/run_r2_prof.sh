# Round-2 evidence: ncu --set full of the scheduler kernel (source-level), keygen / verify kernels,
# launch list of the bench command.  Run under gpurun; outputs to gpurun_out/.
set -e
mkdir -p gpurun_out
export DLB_NO_PEAK=1
T=${T:-r02}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sign_persistent" -c 1 -o gpurun_out/prof_sign_$T -f python scripts/perf_probe.py 2 100000 sign 0 > gpurun_out/ncu_sign.log 2>&1 || (tail -5 gpurun_out/ncu_sign.log; exit 1)
python scripts/ncu_summary.py gpurun_out/prof_sign_$T.ncu-rep gpurun_out/${T}_kernels_sign > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sign_persistent" -c 1 -o gpurun_out/prof_sign1m_$T -f python scripts/perf_probe.py 2 1000000 sign 0 > gpurun_out/ncu_sign1m.log 2>&1 || (tail -5 gpurun_out/ncu_sign1m.log; exit 1)
python scripts/ncu_summary.py gpurun_out/prof_sign1m_$T.ncu-rep gpurun_out/${T}_kernels_sign_1m > /dev/null
timeout 600 ncu --set full --clock-control none -k regex:"k_" -c 80 -o /tmp/prof_kv -f python scripts/perf_probe.py 2 100000 keygen,verify 0 > gpurun_out/ncu_kv.log 2>&1 || (tail -5 gpurun_out/ncu_kv.log; exit 1)
python scripts/ncu_summary.py /tmp/prof_kv.ncu-rep gpurun_out/${T}_kernels_keygen_verify > /dev/null
for lv in 3 5; do
timeout 600 ncu --set full --clock-control none -k regex:"k_sign_persistent" -c 1 -o /tmp/prof_sign_l$lv -f python scripts/perf_probe.py $lv 100000 sign 0 > gpurun_out/ncu_sign$lv.log 2>&1 || (tail -5 gpurun_out/ncu_sign$lv.log; exit 1)
python scripts/ncu_summary.py /tmp/prof_sign_l$lv.ncu-rep gpurun_out/${T}_kernels_sign_l$lv > /dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-levels --no-stream --no-shim > gpurun_out/bench_under_ncu.json 2> gpurun_out/bench_under_ncu.err || (tail -5 gpurun_out/bench_under_ncu.err; exit 1)
ls -la gpurun_out | tail -20
