#!/bin/bash
# A/B of library builds (scripts/build_variant.sh): device-resident rates, builds alternating.
# usage: gpurun -- 'bash scripts/ab_libs.sh <out-name> <levels> <n> <ops> <suffix> [<suffix> ...]'   ("default" = the in-tree build)
out=gpurun_out/$1.txt; lv=$2; n=$3; ops=$4; shift 4
: > $out
for i in 1 2 3; do
  for v in "$@"; do
    lib=paper_2211_12265_b200/libdilithium_b200_$v.so
    [ $v = default ] && lib=paper_2211_12265_b200/libdilithium_b200.so
    echo "== $v run $i" >> $out
    DLB_NO_PEAK=1 DLB_LIB=$PWD/$lib python scripts/perf_probe.py $lv $n $ops 9 >> $out 2>&1
  done
done
cat $out
