T=r02e
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -k "dropout" tests/test_gpu_kernels.py -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_tests.log
timeout -s KILL 400 python bench.py > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
