timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t61.log 2>&1; echo pytest_exit=$? >> gpurun_out/t61.log
timeout -s KILL 300 python tools/gemm_bench.py > gpurun_out/gb61.log 2>&1
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b61.log 2>&1
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b61_c3.log 2>&1
timeout -s KILL 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b61_c4.log 2>&1
