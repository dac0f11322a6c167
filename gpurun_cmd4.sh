timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests.log
timeout -s KILL 600 python bench.py --config C5 --steps 10 --warmup 3 --sim 8 > gpurun_out/c5_n1_sim8.json 2> gpurun_out/c5.err; echo exit=$? >> gpurun_out/c5.err
timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain4.log 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi64ELi0ELi1E -s 300 -c 2 -o gpurun_out/prof_k7 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k7.log 2>&1; echo ncu_exit=$? >> gpurun_out/ncu_k7.log
tail -3 gpurun_out/gpu_tests.log
