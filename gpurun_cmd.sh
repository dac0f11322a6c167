T=r02i
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -k "bf16" -q -p no:cacheprovider > gpurun_out/${T}_bf16.log 2>&1; echo exit=$? >> gpurun_out/${T}_bf16.log
timeout -s KILL 300 python tools/trace_c2.py > gpurun_out/${T}_trace.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout -s KILL 300 $B > gpurun_out/${T}_plain.json 2> gpurun_out/${T}_plain.err && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:recur2_bwd_kernel -c 1 -o gpurun_out/${T}_bwd $B > gpurun_out/${T}_ncu2.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:recur2f_kernel -c 1 -o gpurun_out/${T}_fwd $B > gpurun_out/${T}_ncu3.log 2>&1
