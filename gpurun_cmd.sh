T=r02q
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -k "wavefront or c2_jet_mixed or dropout_full or c3_wavefront" -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python tools/trace_c2.py > gpurun_out/${T}_trace.log 2>&1
timeout -s KILL 400 python bench.py > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
G2="python tools/gemm_one.py 256 8192 2048 0 0 3 128 1"
G7="python tools/gemm_one.py 256 2048 8192 0 1 3 256 8"
timeout -s KILL 120 $G2 > gpurun_out/${T}_g2.log 2>&1 && timeout -s KILL 600 ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 1 -o gpurun_out/${T}_k2 $G2 > gpurun_out/${T}_ncu_k2.log 2>&1
timeout -s KILL 120 $G7 > gpurun_out/${T}_g7.log 2>&1 && timeout -s KILL 600 ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 1 -o gpurun_out/${T}_k7 $G7 > gpurun_out/${T}_ncu_k7.log 2>&1
