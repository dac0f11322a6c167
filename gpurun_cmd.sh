HDP_RECUR_TRACE=1 timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/trace.json 2> gpurun_out/trace.err
grep "hdp trace" gpurun_out/trace.err | tail -5
