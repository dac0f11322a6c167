timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "dynamic or l2 or c1 or c4" > gpurun_out/v7_tests.log 2>&1; echo exit=$? >> gpurun_out/v7_tests.log
timeout -s KILL 400 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v7_c4.json 2> gpurun_out/v7_c4.err
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v7_c2.json 2> gpurun_out/v7_c2.err
