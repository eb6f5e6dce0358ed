set -x
nvidia-smi > /dev/null
timeout 600 python scripts/k1_timing.py weak1 3 > gpurun_out/gpu32_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_tma" -s 2 -c 1 -o gpurun_out/gpu32_k1t_w1 python scripts/k1_timing.py weak1 3 > gpurun_out/gpu32_ncu.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/gpu32_bench_short.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/gpu32_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/gpu32_ncu_launch.log 2>&1
for cfg in q2 q4 proj; do timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e >> gpurun_out/gpu32_bench_cfgs.log 2>&1; done
