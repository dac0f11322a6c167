nvidia-smi topo -m > gpurun_out/v16_topo.txt 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/v16_multi_tests.log 2>&1; echo exit=$? >> gpurun_out/v16_multi_tests.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/v16_c2_n2.json 2> gpurun_out/v16_c2_n2.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v16_c4_n2.json 2> gpurun_out/v16_c4_n2.err
