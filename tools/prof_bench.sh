#!/bin/bash
# Bench line + launch list + one `ncu --set full` capture of the bench's own
# launch shape (per-launch DRAM bytes and instructions for profiles/traffic.json).
#   gpurun -- 'bash tools/prof_bench.sh TAG [bench args...]'
set -u
TAG=${1:-prof}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
WL=${WL:-cfg5}
KRE=${KRE:-wide}
timeout 1800 python bench.py --workload $WL "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
python tools/prof_launch.py --workload $WL ${PFR:+--frames $PFR} > $OUT/launch.json 2> $OUT/launch.err; echo "launch exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --workload $WL --frames ${LFR:-16384} --chunk ${LFR:-16384} --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $OUT/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$KRE --launch-skip ${NCU_SKIP:-0} -c 1 -o $OUT/full \
  python tools/prof_launch.py --workload $WL ${PFR:+--frames $PFR} > $OUT/ncu_full.log 2>&1; echo "ncu full exit $?"
