#!/bin/bash
# compute-sanitizer over every kernel (tools/sanitize.py), one tool after the other.
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh TAG'
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python tools/sanitize.py > $OUT/$tool.log 2>&1
  echo "$tool exit $? ($(grep -c 'SANITIZE-DONE' $OUT/$tool.log) done, $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1))"
done
