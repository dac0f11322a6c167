timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/persist_tests.log 2>&1; echo exit=$? >> gpurun_out/persist_tests.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench12.json 2>> gpurun_out/bench12.err
tail -3 gpurun_out/persist_tests.log
