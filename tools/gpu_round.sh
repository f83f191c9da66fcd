#!/bin/bash
# One gpurun call's worth of evidence: GPU tests, the bench line, the ncu
# launch list of a short bench run and full ncu captures of each best kernel.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [skip-tests]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest.log 2>&1; echo "pytest=$?" >> $OUT/${TAG}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke=$?" >> $OUT/${TAG}_smoke.log
fi
timeout 1500 python bench.py --steps 5 --warmup 3 > $OUT/${TAG}_bench.log 2>&1; echo "bench=$?" >> $OUT/${TAG}_bench.log
cp $OUT/search_r0.jsonl $OUT/${TAG}_search_r0.jsonl 2>/dev/null  # the later runs below reuse the name
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi_after.csv 2>&1
# the sharded path end to end: 2 ranks (sharing this one GPU), headline only
BENCH_NO_SAVE_BEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 2 --warmup 1 --configs none --no-cpu-baseline > $OUT/${TAG}_bench_2rank.log 2>&1
echo "bench2=$?" >> $OUT/${TAG}_bench_2rank.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $OUT/${TAG}_bench_ref_2rank.log 2>&1
echo "ref2=$?" >> $OUT/${TAG}_bench_ref_2rank.log
# launch list (cold-cache, serialised: compare shares, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/${TAG}_launches.csv \
  env BENCH_NO_SAVE_BEST=1 python bench.py --steps 1 --warmup 1 --per-step 16 --configs none --no-cpu-baseline > $OUT/${TAG}_ncu_bench.log 2>&1
for k in axpy axpy_stream gemv sgemm batched sgemm_tc sgemm_tc_x3 sgemm_1024_x3; do
  if [ -f $OUT/best_$k.json ]; then
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:^ispc_[kt] -s 4 -c 1 \
      -o $OUT/${TAG}_prof_$k -f python tools/profile_best.py $k > $OUT/${TAG}_prof_$k.log 2>&1
  fi
done
echo done > $OUT/${TAG}_done.txt
