# A/B: default library vs variants named in $VARIANTS (suffixes), same box, interleaved
cd /root/repo
export DLB_NO_PEAK=1
for rep in 1 2; do
for v in "" $VARIANTS; do
  if [ -z "$v" ]; then unset DLB_LIB; name=default; else export DLB_LIB=$PWD/paper_2211_12265_b200/libdilithium_b200_$v.so; name=$v; fi
  echo "== $name (rep $rep)"; timeout 300 python scripts/perf_probe.py ${LEVELS:-2} ${SIZES:-10000,100000,1000000} sign 5 2>&1 | grep "sign"
done
done
