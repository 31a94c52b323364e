timeout -s KILL 420 python -m pytest tests/test_gpu_attention.py tests/test_gpu_distributed.py -q -m gpu -p no:cacheprovider -x 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t6.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.log 2>&1
UL_FWD_V1=1 timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_v1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2_kernel|bwd_dkdv_kernel|bwd_dq_kernel" -s 3 -c 3 -o gpurun_out/prof_r6 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu6.log 2>&1
tail -3 gpurun_out/t6.log; cat gpurun_out/bench6.log gpurun_out/bench6_v1.log | cut -c1-200
