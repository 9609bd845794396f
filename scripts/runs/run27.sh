cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r27.json 2> gpurun_out/bench_r27.err || tail -20 gpurun_out/bench_r27.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench_r27.json"))
print("value",d["value"],"e2e",d["e2e"]["value"],"frac",d["roofline"]["frac"])
o=d["ops"]
print("verify",o["verify"]["value"],o["verify"]["e2e"],"keygen",o["keygen"]["value"],o["keygen"]["e2e"])
print("lat",o["batch10k_latency_ms"]); print("streamed",o["sign_streamed_1m"]["value"],o["sign_streamed_1m"]["one_context"])
for lv in ("3","5"): print(lv,{k:(v["value"] if isinstance(v,dict) and "value" in v else v) for k,v in o["levels"][lv].items()})
print("cpu",d["cpu_baseline"])
PY
