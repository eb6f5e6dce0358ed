set -x
nvidia-smi > /dev/null
timeout 600 python scripts/k1_timing.py weak1 3 > gpurun_out/gpu26_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_kernel" -s 2 -c 1 -o gpurun_out/gpu26_k1_w1 python scripts/k1_timing.py weak1 3 > gpurun_out/gpu26_ncu.log 2>&1
timeout 600 python scripts/k1_timing.py q4 3 >> gpurun_out/gpu26_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_kernel" -s 2 -c 1 -o gpurun_out/gpu26_k1_q4 python scripts/k1_timing.py q4 3 >> gpurun_out/gpu26_ncu.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/gpu26_bench_short.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/gpu26_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/gpu26_ncu_launch.log 2>&1
