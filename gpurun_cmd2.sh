for f in test_gpu_a2a test_gpu_attention test_gpu_distributed; do
  timeout -s KILL 420 python -m pytest tests/$f.py -v -m gpu -p no:cacheprovider 2>&1 | grep -vE "^$|PASSED" | tail -60 > gpurun_out/$f.log
done
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1
tail -3 gpurun_out/*.log
