set -e
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python scripts/perf_probe.py 2 10000,100000 sign,verify,keygen 5 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err || (tail -5 gpurun_out/bench_r1d.err; exit 1)
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_r1d.json'))
print("sign value %.3fM e2e %.3fM | verify %.3fM e2e %.3fM | verify_shared %.2fM | keygen %.3fM e2e %.3fM"%(d['value']/1e6,d['e2e']['value']/1e6,d['ops']['verify']['value']/1e6,d['ops']['verify']['e2e']/1e6,d['ops']['verify_shared_key']['value']/1e6,d['ops']['keygen']['value']/1e6,d['ops']['keygen']['e2e']/1e6))
print("lat10k", d['ops']['batch10k_latency_ms'], "frac", d['roofline']['frac'], d['roofline']['per_op_frac'])
PY
