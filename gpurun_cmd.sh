HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/trace.json 2> gpurun_out/trace.err
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "persistent or c2 or c3" > gpurun_out/persist_tests.log 2>&1; echo exit=$? >> gpurun_out/persist_tests.log
timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench23.json 2>> gpurun_out/bench23.err
grep "hdp trace" gpurun_out/trace.err | tail -2; tail -2 gpurun_out/persist_tests.log
