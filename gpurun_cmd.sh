T=r02c
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout -s KILL 600 python -m pytest tests/test_gpu_exchange.py "tests/test_gpu_parity.py::test_c2_relu_decision_within_rounding" "tests/test_gpu_parity.py::test_degenerate_shapes" -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_tests.log
timeout -s KILL 120 ./tools/micro/mma_floor > gpurun_out/${T}_mma_floor.txt 2>&1
timeout -s KILL 120 ./tools/micro/push_rt > gpurun_out/${T}_push_rt.txt 2>&1
timeout -s KILL 600 python bench.py --config C5 --sim 8 --sizes 1,16,256,1024 > gpurun_out/${T}_c5_n1.json 2> gpurun_out/${T}_c5_n1.err
timeout -s KILL 600 $TR bench.py --gpus 2 --config C5 > gpurun_out/${T}_c5_n2_fp16.json 2> gpurun_out/${T}_c5_n2_fp16.err
timeout -s KILL 600 $TR bench.py --gpus 2 --config C5 --wire fp32 > gpurun_out/${T}_c5_n2_fp32.json 2> gpurun_out/${T}_c5_n2_fp32.err
timeout -s KILL 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c4_n1.json 2> gpurun_out/${T}_c4_n1.err
timeout -s KILL 600 $TR bench.py --gpus 2 --config C4 --steps 10 --warmup 3 > gpurun_out/${T}_c4_n2.json 2> gpurun_out/${T}_c4_n2.err
timeout -s KILL 600 $TR bench.py --gpus 2 > gpurun_out/${T}_c2_n2.json 2> gpurun_out/${T}_c2_n2.err
