cd /root/repo
export DLB_NO_PEAK=1
for d in 5 8 12 16 31; do
echo "== SPEC_DEPTH=$d"; DLB_SPEC_DEPTH=$d timeout 300 python scripts/perf_probe.py 2 1000,10000,100000,1000000 sign 7 2>&1 | grep sign | cut -c1-100
done
