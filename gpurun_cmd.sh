timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > gpurun_out/t93.log 2>&1; echo pytest_exit=$? >> gpurun_out/t93.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b93.log 2>&1
