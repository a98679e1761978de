#!/bin/bash
# One GPU-box pass: gpu tests, default bench line, ncu launch list of the same
# command.  Usage (from the build container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh TAG'
set -u
TAG=${1:-check}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
cat $OUT/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --frames 8192 --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu.log 2>&1; echo "ncu exit $?"
