timeout -s KILL 300 python tools_timing_ab.py > gpurun_out/ab12.log 2>&1
timeout -s KILL 400 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_distributed.py -q -m gpu -p no:cacheprovider 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t12.log
cat gpurun_out/ab12.log; tail -5 gpurun_out/t12.log
