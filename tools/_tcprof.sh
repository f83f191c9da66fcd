timeout 300 python -m pytest tests/test_gpu_tiles.py -x -q -m gpu -k "tcgen05" > gpurun_out/tc6_pytest.log 2>&1; echo pytest=$? >> gpurun_out/tc6_pytest.log
timeout 600 python tools/tc_variants.py 4096 4096 4096 > gpurun_out/tc6_variants.log 2>&1
