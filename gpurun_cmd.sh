timeout -s KILL 300 python tools/c4_gemm_sweep.py > gpurun_out/v8_sweep.jsonl 2> gpurun_out/v8_sweep.err
timeout -s KILL 300 python tools/gemm_bench.py > gpurun_out/v8_gemm_bench.jsonl 2> gpurun_out/v8_gemm_bench.err
timeout -s KILL 400 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v8_c4.json 2> gpurun_out/v8_c4.err
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x > gpurun_out/v8_tests.log 2>&1; echo exit=$? >> gpurun_out/v8_tests.log
