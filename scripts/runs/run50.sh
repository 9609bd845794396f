cd /root/repo
export DLB_NO_PEAK=1
mkdir -p gpurun_out
timeout 1500 python scripts/parity_campaign.py 300000 990017 2>&1 | tee gpurun_out/parity_run5.txt | tail -5
