cd /root/repo
export DLB_NO_PEAK=1
for cl in 0 3; do echo CONSOLIDATE=$cl; DLB_CONSOLIDATE=$cl timeout 120 python scripts/timeline_probe.py 100000 2 2>&1 | tail -6; done
for cl in 0 1 2 3 4 6; do
echo "== stream CONSOLIDATE=$cl"; DLB_CONSOLIDATE=$cl timeout 120 python scripts/stream_probe.py 1000000 100000 2 2>&1 | grep lanes
done
echo "== single call, CONSOLIDATE=0"; DLB_CONSOLIDATE=0 timeout 120 python scripts/perf_probe.py 2 10000,100000,1000000 sign 5 2>&1 | grep sign | cut -c1-110
