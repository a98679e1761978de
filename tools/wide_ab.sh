#!/bin/bash
# cfg5 wide-kernel env A/B: gpurun -- 'bash tools/wide_ab.sh TAG "NAME:ENV=V,ENV=V" ...'
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
F=${F:-131072}
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}; envs=${envs//,/ }
  env $envs timeout 900 python bench.py --workload cfg5 --frames $F --chunk $F --steps ${STEPS:-1} --warmup 1 --no-e2e --no-cpu \
     > $OUT/$name.json 2> $OUT/$name.err
  echo "$name [$envs] exit $? $(python -c "import json,sys; d=json.load(open('$OUT/$name.json')); print(round(d['value']), round(d['edge_updates_per_s']/1e9,1), round(d['roofline']['frac'],3), d['mean_iterations'])" 2>&1 | tail -1)"
done
