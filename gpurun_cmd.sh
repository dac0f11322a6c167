T=r02f
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout -s KILL 400 python bench.py > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -k "dropout" tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_tests.log
timeout -s KILL 600 $TR bench.py --gpus 2 --config C5 > gpurun_out/${T}_c5_n2_fp16.json 2> gpurun_out/${T}_c5_n2_fp16.err
timeout -s KILL 600 $TR bench.py --gpus 2 --config C5 --wire fp32 > gpurun_out/${T}_c5_n2_fp32.json 2> gpurun_out/${T}_c5_n2_fp32.err
timeout -s KILL 600 $TR bench.py --gpus 2 > gpurun_out/${T}_c2_n2.json 2> gpurun_out/${T}_c2_n2.err
