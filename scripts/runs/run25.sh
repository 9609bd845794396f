cd /root/repo
export DLB_NO_PEAK=1
for mc in 8 32; do
for cl in 0 2 4; do
echo "== MAXCONN=$mc stream CONSOLIDATE=$cl"; CUDA_DEVICE_MAX_CONNECTIONS=$mc DLB_CONSOLIDATE=$cl timeout 120 python scripts/stream_probe.py 1000000 100000 2 2>&1 | grep lanes
done
done
