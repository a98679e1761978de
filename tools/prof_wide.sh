#!/bin/bash
# ncu --set full capture of one wide-kernel launch (cfg5, FR frames) per variant.
#   gpurun -- 'VARS="0 1" bash tools/prof_wide.sh TAG'
set -u
TAG=${1:-profwide}
OUT=gpurun_out/$TAG
mkdir -p $OUT
FR=${FR:-8192}
for v in ${VARS:-0}; do
  ADMM_B200_WIDE_VARIANT=$v python tools/prof_decode.py --code cfg5_n16384 --frames $FR --snr 2.5 > $OUT/plain_$v.log 2>&1; echo "plain $v exit $?"
  ADMM_B200_WIDE_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide -c 1 -o $OUT/wide_$v \
    python tools/prof_decode.py --code cfg5_n16384 --frames $FR --snr 2.5 > $OUT/ncu_$v.log 2>&1; echo "ncu $v exit $?"
done
