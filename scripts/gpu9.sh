set -x
timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu9_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu9_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu9_spmm.log 2>&1; done
for cfg in q4 weak1; do BMV_LIB=$PWD/scratch_libbmv_mb4.so timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu9_k1.log 2>&1; done
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu9_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_chunk|mmult_chunk|tm_reduce" -s 4 -c 4 -o gpurun_out/gpu9_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu9_ncu.log 2>&1
timeout 300 python scripts/k1_timing.py q4 3 > gpurun_out/gpu9_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cellop" -s 2 -c 1 -o gpurun_out/gpu9_k1_q4 python scripts/k1_timing.py q4 3 > gpurun_out/gpu9_ncu2.log 2>&1
