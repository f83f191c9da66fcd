timeout 900 python tools/tc_variants.py 4096 4096 4096 TF32 128,144 4 > gpurun_out/tc11_variants.log 2>&1
timeout 900 python tools/tc_variants.py 4096 4096 4096 TF32 128,144 2 >> gpurun_out/tc11_variants.log 2>&1
