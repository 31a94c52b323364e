for f in test_gpu_attention test_gpu_distributed test_gpu_a2a; do
  timeout -s KILL 420 python -m pytest tests/$f.py -q -m gpu -p no:cacheprovider -x 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/$f.log
done
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_dkdv_kernel|bwd_dq_kernel" -s 2 -c 2 -o gpurun_out/prof_bwd2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/*.log
