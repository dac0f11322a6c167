timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t56.log 2>&1; echo pytest_exit=$? >> gpurun_out/t56.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b56.log 2>&1
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b56_c3.log 2>&1
