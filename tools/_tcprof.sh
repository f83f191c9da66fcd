timeout 300 python -m pytest tests/test_gpu_tiles.py -x -q -m gpu -k "tcgen05" > gpurun_out/tc5_pytest.log 2>&1; echo pytest=$? >> gpurun_out/tc5_pytest.log
timeout 500 python tools/tc_variants.py 4096 4096 4096 TF32 > gpurun_out/tc5_variants.log 2>&1
for v in "s2:staging=SHARED engine=TF32 split=1 bn=256 stages=2" "p2:staging=TMA engine=TF32 split=2 bn=256 stages=4"; do
  tag=${v%%:*}; args=${v#*:}
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:^ispc_t -s 3 -c 1 -o gpurun_out/tc5prof_$tag python tools/profile_tc.py 4096 4096 4096 $args > gpurun_out/tc5prof_$tag.log 2>&1
done
