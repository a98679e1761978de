#!/bin/bash
# Wide-kernel check: streaming GPU tests + cfg5 bench A/B.  gpurun -- 'bash tools/wide_check.sh TAG'
set -u
TAG=${1:-wide}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_streaming.py -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?"; tail -15 $OUT/pytest.log
F=${F:-131072}
run() { # name env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --workload cfg5 --frames $F --chunk $F --steps 1 --warmup 1 --no-e2e --no-cpu \
     > $OUT/$name.json 2> $OUT/$name.err
  echo "$name exit $? $(python -c "import json,sys; d=json.load(open('$OUT/$name.json')); print(round(d['value']), round(d['edge_updates_per_s']/1e9,1), round(d['roofline']['frac'],3), d['roofline']['kernel'])" 2>&1 | tail -1)"
}
run wide
for S in ${SLOTS:-2048 8192}; do run wide_$S ADMM_B200_WIDE_SLOTS=$S; done
run shard ADMM_B200_NO_WIDE=1
