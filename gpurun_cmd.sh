timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/persist_tests.log 2>&1; echo exit=$? >> gpurun_out/persist_tests.log
timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench31.json 2>> gpurun_out/bench31.err
HDP_WAVEFRONT_BC=16 timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench31_bc16.json 2>> gpurun_out/bench31.err
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench31_c3.json 2>> gpurun_out/bench31.err
HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/trace.json 2> gpurun_out/trace.err
tail -2 gpurun_out/persist_tests.log
