#!/bin/bash
# ncu --set full of the resident regular kernel (cfg2, 8192 frames at 1.5 dB)
# and of the cluster kernel on the bench's cfg5 launch shape.
set -u
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resident --launch-skip 1 -c 1 -o $OUT/res \
  python tools/prof_decode.py --code cfg2_n1008 --frames 8192 --snr 1.5 > $OUT/ncu_res.log 2>&1; echo "ncu res exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cluster --launch-skip 1 -c 1 -o $OUT/cluster \
  python tools/prof_launch.py --workload cfg5 ${PFR:+--frames $PFR} > $OUT/ncu_cluster.log 2>&1; echo "ncu cluster exit $?"
