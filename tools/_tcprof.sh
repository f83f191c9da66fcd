timeout 300 python -m pytest tests/test_gpu_tiles.py -x -q -m gpu -k "tcgen05_persistent" > gpurun_out/tc9_pytest.log 2>&1; echo pytest=$? >> gpurun_out/tc9_pytest.log
timeout 900 python tools/tc_variants.py 4096 4096 4096 TF32,TF32X3 148 > gpurun_out/tc9_variants.log 2>&1
