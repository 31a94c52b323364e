timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_distributed.py -q -m gpu -p no:cacheprovider -x 2>&1 | grep -vE "^$" | tail -20 > gpurun_out/t14.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench14.log 2>&1
timeout -s KILL 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|bwd|a2a" --csv --log-file gpurun_out/launches_r14.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/t14.log
