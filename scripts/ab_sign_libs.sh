#!/bin/bash
# A/B of library builds on the signing paths: 1M-task synchronous call (= steady state), key modes.
# usage: gpurun -- 'bash scripts/ab_sign_libs.sh <out-name> <suffix> [<suffix> ...]'   ("default" = in-tree build)
out=gpurun_out/$1.txt; shift
: > $out
for i in 1 2; do
  for v in "$@"; do
    lib=paper_2211_12265_b200/libdilithium_b200_$v.so
    [ $v = default ] && lib=paper_2211_12265_b200/libdilithium_b200.so
    echo "== $v run $i" >> $out
    DLB_NO_PEAK=1 DLB_LIB=$PWD/$lib python scripts/perf_probe.py 2 1000000 sign 3 2>&1 | grep "sign" >> $out
    DLB_LIB=$PWD/$lib python scripts/keymode_probe.py 2 100000 2>&1 | tail -6 >> $out
  done
done
cat $out
