timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02fin_tests.log 2>&1; echo exit=$? >> gpurun_out/r02fin_tests.log
timeout -s KILL 300 python bench.py > gpurun_out/r02fin_c2_n1.json 2> gpurun_out/r02fin_c2_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02fin_c2_n2.json 2> gpurun_out/r02fin_c2_n2.err
timeout -s KILL 300 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r02fin_c3_n1.json 2> gpurun_out/r02fin_c3_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --config C3 --steps 10 --warmup 3 > gpurun_out/r02fin_c3_n2.json 2> gpurun_out/r02fin_c3_n2.err
timeout -s KILL 300 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/r02fin_c4_n1.json 2> gpurun_out/r02fin_c4_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config C4 --steps 3 --warmup 3 > gpurun_out/r02fin_c4_n2.json 2> gpurun_out/r02fin_c4_n2.err
timeout -s KILL 300 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02fin_c5_n1.json 2> gpurun_out/r02fin_c5_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 2 --config C5 --steps 10 --warmup 3 > gpurun_out/r02fin_c5_n2.json 2> gpurun_out/r02fin_c5_n2.err
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02fin_ref.json 2> gpurun_out/r02fin_ref.err
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02fin_smoke.log 2>&1; echo exit=$? >> gpurun_out/r02fin_smoke.log
