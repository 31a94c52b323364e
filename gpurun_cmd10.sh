timeout -s KILL 500 python -m pytest tests/ -q -m gpu -p no:cacheprovider 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t10.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench10.log 2>&1
timeout -s KILL 900 python tools_sweep.py --out gpurun_out/r1_sweep_v2.json > gpurun_out/sweep10.log 2>&1
tail -3 gpurun_out/t10.log
