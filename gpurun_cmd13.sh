timeout -s KILL 600 python -m pytest tests/ -q -m gpu -p no:cacheprovider 2>&1 | grep -vE "^$" | tail -30 > gpurun_out/t13.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench13.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_kernel|bwd_dkdv_kernel|bwd_dq_kernel|a2a_copy" -s 6 -c 4 -o gpurun_out/prof_r13 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu13.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_r13.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
tail -5 gpurun_out/t13.log
