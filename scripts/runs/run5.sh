mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_sv_r1.csv python scripts/perf_probe.py 2 100000 sign,verify 1 > gpurun_out/ncu_probe2.log 2>&1; tail -3 gpurun_out/ncu_probe2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sign_persistent -c 1 -o gpurun_out/prof_sign_r1 -f python scripts/perf_probe.py 2 20000 sign 1 > gpurun_out/ncu_full1.log 2>&1; tail -2 gpurun_out/ncu_full1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_expand_a|k_verify_arith|k_verify_final" -c 3 -o gpurun_out/prof_verify_r1 -f python scripts/perf_probe.py 2 16384 verify 1 > gpurun_out/ncu_full2.log 2>&1; tail -2 gpurun_out/ncu_full2.log
ls -la gpurun_out
