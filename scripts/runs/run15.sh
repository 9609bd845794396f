set -e
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err || (tail -5 gpurun_out/bench_r1f.err; exit 1)
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_r1f.json'))
print("sign %.2fM e2e %.2fM"%(d['value']/1e6,d['e2e']['value']/1e6), d['ops']['batch10k_latency_ms'])
for lv,r in d['ops']['levels'].items():
    print(lv, {k:(round(v['value']/1e6,2), round(v['roofline_frac'],3)) for k,v in r.items() if k in('sign','verify','keygen')}, r['batch10k_latency_ms'])
PY
timeout 600 python scripts/sweep.py --levels 2 --phi 1000,2000,4000,6000,10000,20000,50000,100000,200000 --reps 5 > gpurun_out/sweep_phi_l2.csv 2> gpurun_out/sweep.err || (tail -3 gpurun_out/sweep.err; exit 1)
cat gpurun_out/sweep_phi_l2.csv | grep -E "schema|sign" | cut -d, -f3-13
