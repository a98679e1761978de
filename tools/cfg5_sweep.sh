#!/bin/bash
# cfg5 engine/slot sweep (A/B on one box).  gpurun -- 'bash tools/cfg5_sweep.sh TAG'
set -u
TAG=${1:-cfg5}
OUT=gpurun_out/$TAG
mkdir -p $OUT
F=${F:-131072}
run() { # name env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --workload cfg5 --frames $F --chunk $F --steps 1 --warmup 1 --no-e2e --no-cpu \
     > $OUT/$name.json 2> $OUT/$name.err
  echo "$name exit $? $(python -c "import json,sys; d=json.load(open('$OUT/$name.json')); print(round(d['value']), round(d['edge_updates_per_s']/1e9,1), d['roofline']['frac'])" 2>&1)"
}
run shard
for S in ${SLOTS:-1024 2048 4096 8192}; do run stream_$S ADMM_B200_NO_SHARD=1 ADMM_B200_STREAM_SLOTS=$S; done
