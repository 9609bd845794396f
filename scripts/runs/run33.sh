cd /root/repo
export DLB_NO_PEAK=1
for ch in 8192 16384 32768 65536 131072; do
echo "== CHUNK=$ch"; DLB_CHUNK=$ch timeout 300 python scripts/perf_probe.py 2 100000,400000 keygen,verify 5 2>&1 | grep -E "keygen|verify" | cut -c1-80
done
