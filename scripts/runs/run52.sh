cd /root/repo
export DLB_NO_PEAK=1
for d in 5 8 11 16; do echo "== depth $d"; DLB_SPEC_DEPTH=$d timeout 300 python scripts/perf_probe.py 2 10000,100000,1000000 sign 5 2>&1 | grep sign; done
