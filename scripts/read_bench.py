import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print("value %.2f e2e %.2f frac %.3f spec %.3f | 10x10k %.2f ms | lat10k sign %.2f ms | sync e2e %.2f" % (d["value"]/1e6, d["e2e"]["value"]/1e6, d["roofline"]["frac"], d["ops"]["sign"]["speculative_share"], d["ops"]["sign_10x10k_inflight"]["ms_all_ten"], d["ops"]["batch10k_latency_ms"]["sign"], d["ops"]["sign"]["sync"]["e2e"]/1e6))
