cd /root/repo
export DLB_NO_PEAK=1
timeout 900 python -m pytest tests/test_gpu_keygen_verify.py tests/test_gpu_api_and_scale.py -m gpu -x -q 2>&1 | tail -2
for pc in 8192 16384 32768 65536; do
echo "== PIPE_CHUNK=$pc"; DLB_PIPE_CHUNK=$pc timeout 300 python scripts/e2e_probe.py 100000 2>&1 | tail -1
DLB_PIPE_CHUNK=$pc timeout 300 python scripts/e2e_probe.py 10000 2>&1 | tail -1
done
