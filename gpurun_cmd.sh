timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "persistent or c2" > gpurun_out/persist_tests.log 2>&1; echo exit=$? >> gpurun_out/persist_tests.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo exit=$? >> gpurun_out/bench6.err
timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain6.log 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:recur_fwd -s 2 -c 1 -o gpurun_out/prof_recur python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_recur.log 2>&1; echo ncu_exit=$? >> gpurun_out/ncu_recur.log
tail -3 gpurun_out/persist_tests.log
