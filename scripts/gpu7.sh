set -x
timeout 900 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu7_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu7_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu7_spmm.log 2>&1; done
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu7_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_chunk|mmult_chunk|tm_reduce" -s 3 -c 3 -o gpurun_out/gpu7_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu7_ncu.log 2>&1
