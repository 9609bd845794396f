cd /root/repo
export DLB_NO_PEAK=1
SIZES=100000,1000000 VARIANTS="ku2 ku3" bash scripts/runs/ab.sh
for v in "" ku2 ku3; do
  if [ -z "$v" ]; then unset DLB_LIB; else export DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_$v.so; fi
  echo "== keygen/verify ${v:-default}"; timeout 300 python scripts/perf_probe.py 2 100000 keygen,verify 5 2>&1 | grep -E "keygen|verify" | cut -c1-80
done
