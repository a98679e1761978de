#!/bin/bash
# GPU tests + the quick bench lines (no e2e / cpu legs) of the main workloads.
#   gpurun --timeout 2400 -- 'bash tools/quick_check.sh TAG [workloads...]'
set -u
TAG=${1:-quick}; shift || true
WLS=${@:-cfg5 cfg2 cfg3 cfg4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_projection.py -m gpu -x -q > $OUT/pytest_proj.log 2>&1 || { tail -15 $OUT/pytest_proj.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; rc=$?; echo "pytest exit $rc" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
[ $rc -eq 0 ] || { grep -B 30 "^FAILED\|Error" $OUT/pytest_gpu.log | tail -60; exit 1; }
for wl in $WLS; do
  for dt in ${DTYPES:-f32}; do
    timeout ${BENCH_TIMEOUT:-300} python bench.py --workload $wl --dtype $dt --no-e2e --no-cpu > $OUT/bench_${wl}_$dt.json 2> $OUT/bench_${wl}_$dt.err
    echo "$wl $dt exit $? $(python -c "import json; d=json.load(open('$OUT/bench_${wl}_$dt.json')); print(round(d['value']), round(d.get('edge_updates_per_s',0)/1e9,1), d.get('mean_iterations'), d.get('roofline',{}).get('frac'), d['clocks'])" 2>&1 | tail -1)"
  done
done
