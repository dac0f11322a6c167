timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests.log
timeout -s KILL 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout -s KILL 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/gpu_tests.log
