#!/bin/bash
# ncu --set full capture of the resident regular kernel on cfg2 (8192 frames at 1.5 dB).
set -u
TAG=${1:-profres}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resident --launch-skip 1 -c 1 -o $OUT/res \
  python tools/prof_decode.py --code cfg2_n1008 --frames 8192 --snr 1.5 > $OUT/ncu.log 2>&1; echo "ncu exit $?"
