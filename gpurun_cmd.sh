timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t95.log 2>&1; echo pytest_exit=$? >> gpurun_out/t95.log
HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tr95.log 2>&1
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b95.log 2>&1
