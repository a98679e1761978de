#!/bin/bash
# Quick same-box A/B of library builds on the config-5 bench (512k frames per point, no e2e / cpu legs):
#   gpurun -- 'bash tools/ab_quick.sh libA.so libB.so ...'
for r in 1 2; do for l in "$@"; do
  ADMM_B200_LIB=$l timeout 600 python bench.py --no-e2e --no-cpu --steps 2 --warmup 2 --frames 524288 > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$l', round(d['value']), round(d['edge_updates_per_s']/1e9,1), d['stats_one_step_all_ranks']['iter_sum_correct'], d['config']['engine']['cluster_size'])" || tail -3 /tmp/b.err
done; done
