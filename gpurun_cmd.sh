timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/v47_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/v47_gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v47_smoke.log 2>&1; echo exit=$? >> gpurun_out/v47_smoke.log
timeout -s KILL 400 python bench.py > gpurun_out/v47_c2_default.json 2> gpurun_out/v47_c2_default.err
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v47_c3.json 2> gpurun_out/v47_c3.err
timeout -s KILL 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v47_c4.json 2> gpurun_out/v47_c4.err
