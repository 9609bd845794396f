cd /root/repo
mkdir -p gpurun_out
for tool in memcheck racecheck initcheck; do
timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_probe.py > gpurun_out/sanitizer_$tool.log 2>&1
grep -E "^level|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitizer_$tool.log | sed "s/^/$tool: /"
done
