#!/bin/bash
# Rollout-policy experiments on the axpy 2^26 parity space, 3 seeds each, the
# same evaluation budget; prints the explore summary per run.
#  (1) what a rollout does at a dead end: ISPC_ROLLOUT = restart | deep | ancestor
#  (2) how many decisions the Monte-Carlo tree keeps (--tree-depth)
OUT=${1:-gpurun_out/rollout_experiment.log}
WHAT=${2:-mode}
: > $OUT
run() {
  timeout 300 python -m paper_1904_03383_b200.cli explore axpy --n 67108864 \
    --factors 2,4 2,4,8,16,32,64,128,256,512,1024 --evals 480 "$@" >> $OUT 2>&1
}
if [ "$WHAT" = mode ]; then
  for mode in restart deep ancestor; do
    for seed in 3 5 7; do
      echo "mode=$mode seed=$seed" >> $OUT
      ISPC_ROLLOUT=$mode run --seed $seed
    done
  done
else
  for depth in 12 24 48; do
    for seed in 3 5 7; do
      echo "tree_depth=$depth seed=$seed" >> $OUT
      run --seed $seed --tree-depth $depth
    done
  done
fi
