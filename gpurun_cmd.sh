timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "persistent or c2" > gpurun_out/persist_tests.log 2>&1; echo exit=$? >> gpurun_out/persist_tests.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo exit=$? >> gpurun_out/bench5.err
HDP_PERSISTENT=0 timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench5_nopersist.json 2>> gpurun_out/bench5.err
tail -3 gpurun_out/persist_tests.log
