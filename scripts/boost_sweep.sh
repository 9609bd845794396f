# straggler-boost sweep: pipeline throughput (depth 3 and 8), batch latency, 1M-batch rate
for cfg in "0 4" "24 8" "20 6" "16 4" "12 4" "12 2" "8 2"; do
  set -- $cfg
  export DLB_BOOST_THR=$1 DLB_BOOST_DEPTH=$2
  a=$(python scripts/pipe_probe.py 2 100000 8 24 | tail -1)
  lat=$(python scripts/pipe_probe.py 2 100000 8 24 | grep "^   8 " )
  b=$(python scripts/pipe_probe.py 2 100000 3 24 | tail -1)
  c=$(DLB_NO_PEAK=1 python scripts/perf_probe.py 2 1000000 sign 3 | tail -1)
  echo "thr=$1 depth=$2 | $a | $b | $c"
  echo "     $lat"
done
