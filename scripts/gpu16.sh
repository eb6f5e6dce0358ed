set -x
timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu16_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu16_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu16_spmm.log 2>&1; done
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/gpu16_bench_weak1.log 2>&1
timeout 300 python scripts/spmm_timing.py weak1 3 > gpurun_out/gpu16_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_chunk|mmult_chunk|tm_reduce" -s 6 -c 6 -o gpurun_out/gpu16_w1 python scripts/spmm_timing.py weak1 3 > gpurun_out/gpu16_ncu.log 2>&1
