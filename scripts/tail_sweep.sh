#!/bin/bash
# Rejection-loop tail of a lone batch: CTAs with at most DLB_TAIL_U open tasks speculate up to
# DLB_TAIL_DEPTH instead of the cap of 8.  Device-resident synchronous sign calls, n = 10k and 100k.
# usage: gpurun -- 'bash scripts/tail_sweep.sh [levels]'
out=gpurun_out/r02_tail_sweep.txt
lv=${1:-2}
: > $out
for cfg in "0 0" "2 16" "2 32" "4 16" "4 32" "4 127" "8 16" "8 24" "16 16" "1 127" "3 42"; do
  set -- $cfg
  echo "== DLB_TAIL_U=$1 DLB_TAIL_DEPTH=$2" >> $out
  DLB_NO_PEAK=1 DLB_TAIL_U=$1 DLB_TAIL_DEPTH=$2 python scripts/perf_probe.py $lv 10000,100000 sign 9 >> $out 2>&1
done
cat $out
