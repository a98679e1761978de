#!/bin/bash
# A/B two builds of the library on one box: gpurun -- 'bash tools/ab_lib.sh TAG libA libB [bench args]'
set -u
TAG=$1; A=$2; B=$3; shift 3
OUT=gpurun_out/$TAG
mkdir -p $OUT
for r in 1 2; do
for lib in $A $B; do
  n=$(basename $lib .so)_$r
  ADMM_B200_LIB=$lib timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 2 "$@" > $OUT/$n.json 2> $OUT/$n.err
  echo "$n exit $? $(python -c "import json; d=json.load(open('$OUT/$n.json')); print(round(d['value']), round(d['edge_updates_per_s']/1e9,1), d['mean_iterations'])" 2>&1 | tail -1)"
done
done
