set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/gpu31_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu31_pytest.log
for cfg in q2 proj; do for p in 1 0; do BMV_K1_PAIR=$p timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu31_k1.log 2>&1; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_pair" -s 2 -c 1 -o gpurun_out/gpu31_k1p_q2 python scripts/k1_timing.py q2 3 > gpurun_out/gpu31_ncu.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/gpu31_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu31_pytest_slow.log
