timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/t88_all.log 2>&1; echo pytest_exit=$? >> gpurun_out/t88_all.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/b88_n2.log 2>&1; echo bench_exit=$? >> gpurun_out/b88_n2.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/b88_n1.log 2>&1
