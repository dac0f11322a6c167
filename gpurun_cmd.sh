timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "c2 or c1" > gpurun_out/v44_tests.log 2>&1; echo exit=$? >> gpurun_out/v44_tests.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v44_c2.json 2> gpurun_out/v44_c2.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v44_c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v44_ncu.log 2>&1
