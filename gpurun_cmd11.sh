timeout -s KILL 500 python -m pytest tests/ -q -m gpu -p no:cacheprovider 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t11.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench11.log 2>&1
tail -5 gpurun_out/t11.log
