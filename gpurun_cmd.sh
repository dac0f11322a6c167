timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k7_cluster" > gpurun_out/r02ba_tests.log 2>&1; echo exit=$? >> gpurun_out/r02ba_tests.log
for o in 1 0; do timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --option k7_cluster=$o > gpurun_out/r02ba_c4_k$o.json 2> gpurun_out/r02ba_c4_k$o.err; done
