nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02b_smi.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_exchange.py -q -p no:cacheprovider > gpurun_out/r02b_exchange.log 2>&1; echo exit=$? >> gpurun_out/r02b_exchange.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 --deselect tests/test_gpu_exchange.py > gpurun_out/r02b_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/r02b_gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo exit=$? >> gpurun_out/r02b_smoke.log
timeout -s KILL 400 python bench.py > gpurun_out/r02b_c2.json 2> gpurun_out/r02b_c2.err
timeout -s KILL 400 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02b_c3.json 2> gpurun_out/r02b_c3.err
