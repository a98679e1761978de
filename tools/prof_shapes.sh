#!/bin/bash
# ncu --set full of the bench launch shape of several workloads; keeps only the
# text summaries (the reports would exceed gpurun's copy-back limit).
#   gpurun -- 'bash tools/prof_shapes.sh TAG "cfg3 f32" "cfg4 f32" ...'
set -u
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for spec in "$@"; do
  set -- $spec; wl=$1; dt=$2
  python tools/prof_launch.py --workload $wl --dtype $dt > $O/launch_${wl}_$dt.json 2>/dev/null
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-resident} --launch-skip 1 -c 1 -o /tmp/rep_${wl}_$dt \
    python tools/prof_launch.py --workload $wl --dtype $dt > $O/ncu_${wl}_$dt.log 2>&1
  echo "$wl $dt ncu $?"
  python tools/ncu_summary.py /tmp/rep_${wl}_$dt.ncu-rep --lines 12 > $O/ncu_${wl}_$dt.txt 2>&1
  rm -f /tmp/rep_${wl}_$dt.ncu-rep
done
