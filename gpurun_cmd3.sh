timeout -s KILL 400 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_attention.py -v -m gpu -p no:cacheprovider -k "fp32 or golden or config1" 2>&1 | grep -vE "^$|PASSED" | tail -40 > gpurun_out/t3.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_kernel|bwd_dkdv_kernel|bwd_dq_kernel" -s 3 -c 3 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/t3.log; ls -la gpurun_out
