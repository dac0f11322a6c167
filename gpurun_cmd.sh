timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wavefront_matches or pdl or c2_full" > gpurun_out/r02ay_tests.log 2>&1; echo exit=$? >> gpurun_out/r02ay_tests.log
timeout 300 python bench.py > gpurun_out/r02ay_c2.json 2> gpurun_out/r02ay_c2.err
