cd /root/repo
export DLB_NO_PEAK=1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python scripts/perf_probe.py 2,44,65,87 100000 keygen,sign,verify 5 2>&1 | grep -E "sign|keygen|verify" | cut -c1-100
