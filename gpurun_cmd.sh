T=r02d
timeout -s KILL 300 python tools/c4_multicast_sweep.py > gpurun_out/${T}_mc_sweep.jsonl 2> gpurun_out/${T}_mc_sweep.err
timeout -s KILL 900 python -m pytest tests/test_gpu_convergence.py -q -p no:cacheprovider > gpurun_out/${T}_conv.log 2>&1; echo exit=$? >> gpurun_out/${T}_conv.log
cp gpurun_out/convergence_auc.json gpurun_out/${T}_convergence_auc.json 2>/dev/null
