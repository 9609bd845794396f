cd /root/repo
export DLB_NO_PEAK=1
for co in -1 100 75 50 25; do
echo "== CARVEOUT=$co"; DLB_CARVEOUT=$co timeout 300 python scripts/perf_probe.py 2 100000 keygen,verify 5 2>&1 | grep -E "keygen|verify" | cut -c1-80
done
