T=r02g
timeout -s KILL 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > gpurun_out/${T}_gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo exit=$? >> gpurun_out/${T}_smoke.log
cp gpurun_out/parity_errors.jsonl gpurun_out/${T}_parity_errors.jsonl 2>/dev/null
