cd /root/repo
export DLB_NO_PEAK=1 DLB_SPEC_DEPTH=8
for pad in 0 17000 30000 60000; do
echo "== PAD=$pad"; DLB_SIGN_PAD_SMEM=$pad timeout 300 python scripts/perf_probe.py 2 100000,1000000 sign 3 2>&1 | tail -2
done
