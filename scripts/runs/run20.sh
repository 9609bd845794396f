cd /root/repo
export DLB_NO_PEAK=1
for d in 0 1 2 3 5 8 65535; do
echo "== SPEC_DEPTH=$d"; DLB_SPEC_DEPTH=$d timeout 300 python scripts/perf_probe.py 2 10000,100000,1000000 sign 5 2>&1 | tail -3
done
echo "== MONT_WIDE"; DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_mw.so timeout 300 python scripts/perf_probe.py 2 100000,1000000 sign,verify,keygen 5 2>&1 | tail -6
echo "== base all ops"; timeout 300 python scripts/perf_probe.py 2 100000,1000000 sign,verify,keygen 5 2>&1 | tail -6
