cd /root/repo
mkdir -p gpurun_out
timeout 900 python scripts/sweep.py --levels 2,3,5 --phi 1000,10000,100000 --psi 0 --reps 7 > gpurun_out/r01c_sweep.csv 2> gpurun_out/sweep.err || tail -5 gpurun_out/sweep.err
cat gpurun_out/r01c_sweep.csv | head -40
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r01c_bench.json 2> gpurun_out/r01c_bench.err || tail -5 gpurun_out/r01c_bench.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/r01c_bench.json"))
print("value",d["value"],"e2e",d["e2e"]["value"],"frac",d["roofline"]["frac"])
for lv,r in d["ops"]["levels"].items(): print(lv,{k:round(v["value"]) for k,v in r.items() if isinstance(v,dict) and "value" in v}, r["batch10k_latency_ms"])
PY
