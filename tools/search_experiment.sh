#!/bin/bash
# Search-policy experiment on the axpy 2^26 parity space: each setting runs the
# same 480-evaluation explore with seeds 1..8 (the multi-threaded pipeline is
# not reproducible run to run, so one seed says little); prints one summary
# line per run. Settings: environment knobs of host/search.cpp + tree depth.
OUT=${1:-gpurun_out/search_experiment.log}
shift
SETTINGS=("$@")
[ ${#SETTINGS[@]} -eq 0 ] && SETTINGS=("ISPC_GREEDY=random:48" "ISPC_GREEDY=random ISPC_GREEDY_P=0.75:48" \
  "ISPC_GREEDY=random:96" "ISPC_GREEDY=random ISPC_GREEDY_P=0.75:96")
: > $OUT
for s in "${SETTINGS[@]}"; do
  envs=${s%%:*}; depth=${s##*:}
  for seed in 1 2 3 4 5 6 7 8; do
    echo "setting=$s seed=$seed" >> $OUT
    env $envs timeout 120 python -m paper_1904_03383_b200.cli explore axpy --n 67108864 \
      --factors 2,4 2,4,8,16,32,64,128,256,512,1024 --evals 480 --seed $seed --tree-depth $depth >> $OUT 2>&1
  done
done
