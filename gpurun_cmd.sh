timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wavefront or c2" > gpurun_out/t45.log 2>&1; echo pytest_exit=$? >> gpurun_out/t45.log
for fx in 1 0; do
HDP_WAVEFRONT_FUSEX=$fx HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tr45_$fx.log 2>&1
HDP_WAVEFRONT_FUSEX=$fx timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b45_$fx.log 2>&1
done
