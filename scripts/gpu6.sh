set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu6_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu6_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu6_spmm.log 2>&1; done
timeout 600 python bench.py --config q4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gpu6_bench_q4.log 2>&1
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu6_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_chunk|mmult_chunk|tm_reduce" -s 3 -c 3 -o gpurun_out/gpu6_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu6_ncu.log 2>&1
