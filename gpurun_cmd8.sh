timeout -s KILL 420 python -m pytest tests/test_gpu_attention.py tests/test_gpu_distributed.py -q -m gpu -p no:cacheprovider -x 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t8.log
timeout -s KILL 120 python tools_e2e_diag.py > gpurun_out/diag8.log 2>&1
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.log 2>&1
tail -3 gpurun_out/t8.log; cat gpurun_out/diag8.log; cat gpurun_out/bench8.log | cut -c1-200
