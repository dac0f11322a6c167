timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/v13_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/v13_gpu_tests.log
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v13_c3.json 2> gpurun_out/v13_c3.err
