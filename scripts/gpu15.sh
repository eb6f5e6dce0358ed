set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu15_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu15_pytest.log
for cfg in q2 q4 weak1; do
  timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu15_k1.log 2>&1
  BMV_LIB=$PWD/scratch_mb2.so timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu15_k1.log 2>&1
  BMV_LIB=$PWD/scratch_prev.so timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu15_k1.log 2>&1
done
