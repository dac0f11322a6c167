timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/v15_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/v15_gpu_tests.log
timeout -s KILL 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v15_c4.json 2> gpurun_out/v15_c4.err
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v15_c3.json 2> gpurun_out/v15_c3.err
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/v15_c2.json 2> gpurun_out/v15_c2.err
