cd /root/repo
export DLB_NO_PEAK=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_primitives.py -m gpu -x -q 2>&1 | tail -2
timeout 1500 python scripts/parity_campaign.py 300000 424242 2>&1 | tee gpurun_out/parity_run4.txt | tail -5
