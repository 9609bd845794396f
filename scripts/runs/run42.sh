cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for tool in memcheck racecheck initcheck; do
timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_probe.py > gpurun_out/sanitizer_$tool.log 2>&1
grep -E "^level|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitizer_$tool.log | sed "s/^/$tool: /"
done
bash scripts/runs/run28.sh 2>&1 | tail -2
