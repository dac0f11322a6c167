timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "head_fused" > gpurun_out/r02az_tests.log 2>&1; echo exit=$? >> gpurun_out/r02az_tests.log
