set -x
timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu12_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu12_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu12_spmm.log 2>&1; done
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu12_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_chunk|mmult_chunk" -s 3 -c 3 -o gpurun_out/gpu12_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu12_ncu.log 2>&1
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu12_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mmult_chunk" -s 2 -c 2 -o gpurun_out/gpu12_mm_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu12_ncu2.log 2>&1
