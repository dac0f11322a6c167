T=r02j
timeout -s KILL 300 python tools/trace_c2.py > gpurun_out/${T}_trace.log 2>&1
timeout -s KILL 300 python tools/trace_c2.py 64 128 > gpurun_out/${T}_trace_b64.log 2>&1
