#!/bin/bash
# cfg5 wide-kernel variant A/B: gpurun -- 'VARS="0 1 3" bash tools/wide_var.sh TAG'
set -u
TAG=${1:-widevar}
OUT=gpurun_out/$TAG
mkdir -p $OUT
F=${F:-131072}
run() { # name env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --workload cfg5 --frames $F --chunk $F --steps 1 --warmup 1 --no-e2e --no-cpu \
     > $OUT/$name.json 2> $OUT/$name.err
  echo "$name exit $? $(python -c "import json,sys; d=json.load(open('$OUT/$name.json')); print(round(d['value']), round(d['edge_updates_per_s']/1e9,1), round(d['roofline']['frac'],3), d['roofline']['kernel'])" 2>&1 | tail -1)"
}
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest.log
fi
for v in ${VARS:-0}; do run var_$v ADMM_B200_WIDE_VARIANT=$v ${EXTRA:-}; done
