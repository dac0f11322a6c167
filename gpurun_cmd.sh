timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02fin4_tests.log 2>&1; echo exit=$? >> gpurun_out/r02fin4_tests.log
timeout 300 python bench.py > gpurun_out/r02fin4_c2.json 2> gpurun_out/r02fin4_c2.err
