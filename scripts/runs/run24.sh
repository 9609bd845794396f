cd /root/repo
export DLB_NO_PEAK=1
timeout 300 python -m pytest tests/test_gpu_sign.py -m gpu -x -q 2>&1 | tail -2
for cl in 0 1 2 3 4 6; do
echo "== CONSOLIDATE=$cl"; DLB_CONSOLIDATE=$cl timeout 120 python scripts/perf_probe.py 2 10000,100000 sign 5 2>&1 | grep sign | cut -c1-110
done
for cl in 0 2 4; do
echo "== stream CONSOLIDATE=$cl"; DLB_CONSOLIDATE=$cl timeout 120 python scripts/stream_probe.py 1000000 100000 2 2>&1 | grep lanes
done
