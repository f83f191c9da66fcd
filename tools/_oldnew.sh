OUT=gpurun_out/oldnew.log
: > $OUT
for which in old new; do
  for seed in 1 2 3 4 5 6 7 8; do
    echo "setting=$which seed=$seed" >> $OUT
    if [ $which = old ]; then d=_old; else d=.; fi
    (cd $d && timeout 120 python -m paper_1904_03383_b200.cli explore axpy --n 67108864 \
      --factors 2,4 2,4,8,16,32,64,128,256,512,1024 --evals 480 --seed $seed) >> $OUT 2>&1
  done
done
