timeout -s KILL 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1; echo exit=$? >> gpurun_out/gemm_bench.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "c3" > gpurun_out/c3_tests.log 2>&1; echo exit=$? >> gpurun_out/c3_tests.log
timeout -s KILL 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -3 gpurun_out/c3_tests.log
