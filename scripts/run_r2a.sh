for occ in 4 3 2; do
echo "== DLB_SIGN_OCC=$occ"
DLB_SIGN_OCC=$occ python scripts/async_timeline.py 2 100000 4 2>&1 | tail -5
DLB_SIGN_OCC=$occ python scripts/async_timeline.py 2 10000 10 2>&1 | head -1
DLB_SIGN_OCC=$occ python scripts/async_probe.py 2 2
done
