timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x -k "c4_full or k7_cluster or gemm" > gpurun_out/r02bb_tests.log 2>&1; echo exit=$? >> gpurun_out/r02bb_tests.log
timeout 300 python bench.py > gpurun_out/r02bb_c2.json 2> gpurun_out/r02bb_c2.err
