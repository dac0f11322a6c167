timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x -k "k7_cluster or adam or update" > gpurun_out/r02fin2_tests.log 2>&1; echo exit=$? >> gpurun_out/r02fin2_tests.log
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02fin_c5_n1.json 2> gpurun_out/r02fin_c5_n1.err
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --sim 8 > gpurun_out/r02fin_c5_n1_sim8.json 2> gpurun_out/r02fin_c5_n1_sim8.err
