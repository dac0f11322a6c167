timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/v48_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/v48_gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v48_smoke.log 2>&1; echo exit=$? >> gpurun_out/v48_smoke.log
timeout -s KILL 400 python bench.py > gpurun_out/v48_c2_default.json 2> gpurun_out/v48_c2_default.err
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v48_c2_reference.json 2> gpurun_out/v48_c2_reference.err
