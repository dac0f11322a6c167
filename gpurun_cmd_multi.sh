timeout -s KILL 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02last_tests.log 2>&1; echo exit=$? >> gpurun_out/r02last_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02last_smoke.log 2>&1; echo exit=$? >> gpurun_out/r02last_smoke.log
timeout -s KILL 300 python bench.py > gpurun_out/r02last_c2_n1.json 2> gpurun_out/r02last_c2_n1.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/r02last_c2_n2.json 2> gpurun_out/r02last_c2_n2.err
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/r02last_ref.json 2> gpurun_out/r02last_ref.err
