set -x
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu14_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu14_pytest.log
for cfg in q2 q4 weak1; do timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu14_k1.log 2>&1; BMV_LIB=$PWD/scratch_wide.so timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu14_k1.log 2>&1; done
for cfg in q4 weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu14_spmm.log 2>&1; done
timeout 300 python scripts/k1_timing.py q4 3 > gpurun_out/gpu14_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cellop" -s 2 -c 1 -o gpurun_out/gpu14_k1_q4 python scripts/k1_timing.py q4 3 > gpurun_out/gpu14_ncu.log 2>&1
