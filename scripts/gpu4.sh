set -x
timeout 900 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu4_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu4_pytest.log
for cfg in q2 q4 proj; do timeout 300 python scripts/k1_timing.py $cfg 20 >> gpurun_out/gpu4_k1.log 2>&1; done
timeout 600 python bench.py --config q4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gpu4_bench_q4.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/gpu4_bench_weak1.log 2>&1
timeout 300 python scripts/k1_timing.py q4 5 > gpurun_out/gpu4_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cellop_kernel -s 3 -c 1 -o gpurun_out/gpu4_k1_q4 python scripts/k1_timing.py q4 5 > gpurun_out/gpu4_ncu.log 2>&1
