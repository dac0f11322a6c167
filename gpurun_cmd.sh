timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "persistent or c2 or c3 or c1" > gpurun_out/persist_tests.log 2>&1; echo exit=$? >> gpurun_out/persist_tests.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench10.json 2>> gpurun_out/bench10.err
HDP_RECUR_CLUSTER=0 timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench10_nocl.json 2>> gpurun_out/bench10.err
tail -3 gpurun_out/persist_tests.log
