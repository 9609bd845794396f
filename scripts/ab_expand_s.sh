#!/bin/bash
# A/B of ExpandS's early exit (samplers.cuh, -DDLB_EXPAND_S_NO_EARLY_EXIT): device-resident keygen
# rate at n = 100,000 for levels 2 / 3 / 5, both builds alternating, then the keygen parity tests.
# usage: gpurun -- 'bash scripts/ab_expand_s.sh'   (needs libdilithium_b200_noee.so from build_variant.sh)
out=gpurun_out/r02_expand_s_ab.txt
: > $out
for i in 1 2 3; do
  for v in default noee; do
    lib=paper_2211_12265_b200/libdilithium_b200.so
    [ $v = noee ] && lib=paper_2211_12265_b200/libdilithium_b200_noee.so
    echo "== $v run $i" >> $out
    DLB_NO_PEAK=1 DLB_LIB=$PWD/$lib python scripts/perf_probe.py 2,3,5 100000 keygen 9 >> $out 2>&1
  done
done
python -m pytest tests/test_gpu_keygen_verify.py tests/test_gpu_api_and_scale.py tests/test_gpu_mldsa.py -m gpu -x -q 2>&1 | tail -3 >> $out
cat $out
