set -e
cd /root/repo
mkdir -p gpurun_out
export DLB_NO_PEAK=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sign_persistent" -c 1 -o gpurun_out/prof_sign_r2a -f python scripts/perf_probe.py 2 100000 sign 0 > gpurun_out/ncu_sign.log 2>&1 || (tail -5 gpurun_out/ncu_sign.log; exit 1)
ls -la gpurun_out
