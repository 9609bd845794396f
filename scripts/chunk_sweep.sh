#!/bin/bash
# Device chunk size of keygen / verify (DLB_CHUNK, tasks per ExpandA + arithmetic launch pair): does a
# chunk whose expanded matrices fit the 126 MB L2 (16 KB per Dilithium2 key) beat the 65,536 default?
# usage: gpurun -- 'bash scripts/chunk_sweep.sh'
out=gpurun_out/r02_chunk_sweep.txt
: > $out
for ch in 2048 3072 4096 6144 8192 16384 65536; do
  echo "== DLB_CHUNK=$ch" >> $out
  DLB_NO_PEAK=1 DLB_CHUNK=$ch python scripts/perf_probe.py 2,3,5 100000 keygen 9 >> $out 2>&1
done
cat $out
