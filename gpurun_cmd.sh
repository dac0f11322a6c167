T=r02m
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout -s KILL 300 python tools/trace_c2.py > gpurun_out/${T}_trace.log 2>&1
timeout -s KILL 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/${T}_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_gpu_tests.log
cp gpurun_out/parity_errors.jsonl gpurun_out/${T}_parity_errors.jsonl 2>/dev/null
timeout -s KILL 400 python bench.py > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_c2_ref.json 2> gpurun_out/${T}_c2_ref.err
timeout -s KILL 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
timeout -s KILL 600 $TR bench.py --gpus 2 > gpurun_out/${T}_c2_n2.json 2> gpurun_out/${T}_c2_n2.err
timeout -s KILL 600 $TR bench.py --gpus 2 --config C3 > gpurun_out/${T}_c3_n2.json 2> gpurun_out/${T}_c3_n2.err
timeout -s KILL 600 $TR bench.py --gpus 2 --config C4 --steps 10 --warmup 3 > gpurun_out/${T}_c4_n2.json 2> gpurun_out/${T}_c4_n2.err
