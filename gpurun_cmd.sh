T=r02p
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
nvidia-smi topo -m > gpurun_out/${T}_topo.txt 2>&1
timeout -s KILL 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/${T}_multi4.log 2>&1; echo exit=$? >> gpurun_out/${T}_multi4.log
timeout -s KILL 600 $TR bench.py --gpus 4 > gpurun_out/${T}_c2_n4.json 2> gpurun_out/${T}_c2_n4.err
timeout -s KILL 600 $TR bench.py --gpus 4 --config C3 > gpurun_out/${T}_c3_n4.json 2> gpurun_out/${T}_c3_n4.err
timeout -s KILL 600 $TR bench.py --gpus 4 --config C4 --steps 10 --warmup 3 > gpurun_out/${T}_c4_n4.json 2> gpurun_out/${T}_c4_n4.err
timeout -s KILL 600 $TR bench.py --gpus 4 --config C5 > gpurun_out/${T}_c5_n4_fp16.json 2> gpurun_out/${T}_c5_n4_fp16.err
timeout -s KILL 600 $TR bench.py --gpus 4 --config C5 --wire fp32 > gpurun_out/${T}_c5_n4_fp32.json 2> gpurun_out/${T}_c5_n4_fp32.err
timeout -s KILL 400 python bench.py > gpurun_out/${T}_c2_n1.json 2> gpurun_out/${T}_c2_n1.err
