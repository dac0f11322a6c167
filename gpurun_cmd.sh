T=r02o
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -k "wavefront or c2_jet_mixed or c3_imdb_full or persistent or dropout_full or c3_wavefront or degenerate" -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo exit=$? >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python tools/trace_c2.py > gpurun_out/${T}_trace.log 2>&1
timeout -s KILL 400 python bench.py > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout -s KILL 400 python bench.py --config C3 --no-cpu-baseline > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
