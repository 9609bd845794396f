cd /root/repo
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck python scripts/sanitize_probe.py > gpurun_out/sanitizer_racecheck.log 2>&1
grep -E "^level|RACECHECK SUMMARY" gpurun_out/sanitizer_racecheck.log
grep -E "Warning|Error" gpurun_out/sanitizer_racecheck.log | cut -c1-140 | head -5
