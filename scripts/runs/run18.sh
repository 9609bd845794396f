set -e
cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err || (tail -20 gpurun_out/bench_r18.err; exit 1)
cat gpurun_out/bench_r18.json | head -c 1500
