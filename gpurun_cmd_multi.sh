timeout -s KILL 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/r02z_multi_tests.log 2>&1; echo exit=$? >> gpurun_out/r02z_multi_tests.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r02z_c2_n1.json 2> gpurun_out/r02z_c2_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02z_c2_n2.json 2> gpurun_out/r02z_c2_n2.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02z_c4_n2.json 2> gpurun_out/r02z_c4_n2.err
timeout -s KILL 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02z_c4_n1.json 2> gpurun_out/r02z_c4_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02z_c3_n2.json 2> gpurun_out/r02z_c3_n2.err
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02z_c3_n1.json 2> gpurun_out/r02z_c3_n1.err
