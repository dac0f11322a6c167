timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab54_new.log 2>&1
HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab54_new_tr.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "wavefront or c2" > gpurun_out/t54.log 2>&1; echo pytest_exit=$? >> gpurun_out/t54.log
