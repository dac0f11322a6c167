timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/overlap_timeline.py C4 > gpurun_out/r02an_c4.log 2>&1
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 tools/overlap_timeline.py C2 > gpurun_out/r02an_c2.log 2>&1
timeout -s KILL 300 python tools/overlap_timeline.py C2 > gpurun_out/r02an_c2_n1.log 2>&1
