set -x
timeout 1200 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu8_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu8_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu8_spmm.log 2>&1; done
for cfg in q4 weak1; do BMV_LIB=scratch_libbmv_mb4.so timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu8_k1.log 2>&1; timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu8_k1.log 2>&1; done
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu8_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_chunk|mmult_chunk|tm_reduce|cellop" -s 1 -c 4 -o gpurun_out/gpu8_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu8_ncu.log 2>&1
