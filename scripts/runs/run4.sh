mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo "rc=$?"; tail -5 gpurun_out/bench_r1.err; cat gpurun_out/bench_r1.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r1.json 2>> gpurun_out/bench_r1.err; cat gpurun_out/bench_ref_r1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r1.csv python scripts/perf_probe.py 2 100000 > gpurun_out/ncu_probe.log 2>&1; tail -3 gpurun_out/ncu_probe.log
