#!/bin/bash
# Headline bench A/B of the rollout mode at a dead end (restart vs deep), two
# runs each, configs and CPU baseline skipped (bench lines to $1).
OUT=${1:-gpurun_out/rollout_ab.log}
: > $OUT
for rep in 1 2; do
  for mode in restart deep; do
    echo -n "mode=$mode " >> $OUT
    ISPC_ROLLOUT=$mode BENCH_NO_SAVE_BEST=1 timeout 400 python bench.py --steps 5 --warmup 3 --configs none \
      --no-cpu-baseline --uniform-evals 0 2>/dev/null | tail -1 >> $OUT
  done
done
