timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wavefront or c2 or c3" > gpurun_out/t69.log 2>&1; echo pytest_exit=$? >> gpurun_out/t69.log
HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tr69.log 2>&1
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b69.log 2>&1
