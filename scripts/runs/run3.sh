nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python scripts/perf_probe.py 2 1000,10000,100000 2>&1 | tail -30
