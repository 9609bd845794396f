cd /root/repo
mkdir -p gpurun_out
export DLB_NO_PEAK=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1500 compute-sanitizer --tool initcheck python scripts/sanitize_probe.py > gpurun_out/sanitizer_initcheck.log 2>&1
grep -E "^level|ERROR SUMMARY" gpurun_out/sanitizer_initcheck.log
LEVELS=2,3,5 SIZES=100000 VARIANTS=prev bash scripts/runs/ab.sh
SIZES=10000,1000000 VARIANTS=prev bash scripts/runs/ab.sh
for v in "" prev; do
  if [ -z "$v" ]; then unset DLB_LIB; else export DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_$v.so; fi
  echo "== keygen/verify ${v:-default}"; timeout 300 python scripts/perf_probe.py 2,3,5 100000 keygen,verify 5 2>&1 | grep -E "keygen|verify" | cut -c1-80
done
