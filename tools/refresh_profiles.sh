#!/bin/bash
# Refresh the bench lines of every BASELINE workload, the reference arm, the
# launch lists and the ncu capture of the headline launch shape.
#   gpurun --timeout 3000 -- 'bash tools/refresh_profiles.sh TAG'
set -u
TAG=${1:-refresh}
OUT=gpurun_out/$TAG
mkdir -p $OUT
b() { # name args...
  local name=$1; shift
  timeout 1200 python bench.py "$@" > $OUT/bench_$name.json 2> $OUT/bench_$name.err
  echo "$name exit $? $(python -c "import json; d=json.load(open('$OUT/bench_$name.json')); print(round(d['value']), round(d.get('edge_updates_per_s',0)/1e9,1), d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d['clocks'])" 2>&1 | tail -1)"
}
b cfg5
b cfg2 --workload cfg2
b cfg2_f64 --workload cfg2 --dtype f64
b cfg3 --workload cfg3
b cfg4 --workload cfg4
b cfg1 --workload cfg1 --dtype f64
b cfg1_f32 --workload cfg1
b cfg5_f64 --workload cfg5 --dtype f64 --steps 1 --warmup 3
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/bench_ref_cfg5.json 2> $OUT/bench_ref_cfg5.err; echo "ref exit $?"
python tools/cluster_check.py --frames 8192 > $OUT/cluster_vs_wide.txt 2>&1; echo "cluster_check exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg5.csv \
  python bench.py --frames 16384 --chunk 16384 --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_l5.log 2>&1; echo "ncu cfg5 exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv \
  python bench.py --workload cfg2 --frames 8192 --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_l2.log 2>&1; echo "ncu cfg2 exit $?"
python tools/prof_launch.py --workload cfg5 > $OUT/launch_cfg5.json 2> $OUT/launch_cfg5.err; echo "launch exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cluster --launch-skip 1 -c 1 -o $OUT/cluster_cfg5 \
  python tools/prof_launch.py --workload cfg5 > $OUT/ncu_full_cluster.log 2>&1; echo "ncu full cluster exit $?"
python tools/prof_launch.py --workload cfg2 > $OUT/launch_cfg2.json 2> $OUT/launch_cfg2.err; echo "launch cfg2 exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:resident --launch-skip 1 -c 1 -o $OUT/resident_cfg2 \
  python tools/prof_launch.py --workload cfg2 > $OUT/ncu_full_resident.log 2>&1; echo "ncu full resident exit $?"
