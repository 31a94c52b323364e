timeout -s KILL 420 python -m pytest tests/ -q -m gpu -p no:cacheprovider -x 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t7.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench7.log 2>&1
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.log 2>&1
tail -3 gpurun_out/t7.log; cat gpurun_out/bench7.log | cut -c1-300; cat gpurun_out/smoke7.log
