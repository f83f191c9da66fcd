mkdir -p gpurun_out/axlogs
for seed in 1 2 3 4 5 6; do
  timeout 120 python -m paper_1904_03383_b200.cli explore axpy --n 67108864 \
    --factors 2,4 2,4,8,16,32,64,128,256,512,1024 --evals 600 --seed $seed --log gpurun_out/axlogs/s$seed.jsonl > gpurun_out/axlogs/s$seed.out 2>&1
done
