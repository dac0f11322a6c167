T=r02h
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -k "bf16" -q -p no:cacheprovider > gpurun_out/${T}_bf16.log 2>&1; echo exit=$? >> gpurun_out/${T}_bf16.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_small.py perstep > gpurun_out/${T}_memcheck_perstep.log 2>&1; echo exit=$? >> gpurun_out/${T}_memcheck_perstep.log
