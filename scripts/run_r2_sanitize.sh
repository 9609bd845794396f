# compute-sanitizer passes over the end-to-end probe + the mapping A/B microbenchmark
mkdir -p gpurun_out
out=gpurun_out/${T:-r02}_compute_sanitizer.txt
echo "command: compute-sanitizer --tool {memcheck,racecheck,initcheck} python scripts/sanitize_probe.py (keygen+sign+verify, levels 2/3/5 and ML-DSA-65 incl. a context string; per-task, shared and table-indexed keys; four batches in flight waited out of order; assignment log; bounded attempts)" > $out
for tool in memcheck racecheck initcheck; do
  DLB_SLOW_WARM=1 timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_probe.py 2>&1 | grep -E "ok, mean|SUMMARY|ERROR|Error|hazard" | sed "s/^/$tool: /" >> $out
done
cat $out
build_ab/mapping_ab > gpurun_out/${T:-r02}_mapping_ab.txt; cat gpurun_out/${T:-r02}_mapping_ab.txt
