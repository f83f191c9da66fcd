#!/bin/bash
# Decision-order experiment on the axpy 2^26 parity space (PAPER.md 5.4:
# the order of decisions changes how much the bound prunes). Each order gets
# the same evaluation budget and seed; prints the best kernel per order.
OUT=${1:-gpurun_out/order_experiment.log}
: > $OUT
for ord in "size,dim_kind,thread_level,mem_space,order,cache" \
           "order,size,dim_kind,thread_level,mem_space,cache" \
           "dim_kind,order,size,thread_level,mem_space,cache" \
           "mem_space,order,dim_kind,size,thread_level,cache"; do
  echo "order=$ord" >> $OUT
  timeout 300 python -m paper_1904_03383_b200.cli explore axpy --n 67108864 --factors 2,4 2,4,8,16,32,64,128,256,512,1024 \
    --evals 384 --seed 7 --decision-order "$ord" >> $OUT 2>&1
done
