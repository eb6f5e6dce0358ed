set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/gpu34_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu34_pytest.log
for cfg in q4 weak1; do for c in smem global; do BMV_K1_COEF=$c timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu34_k1.log 2>&1; done; done
BMV_K1_COEF=global timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_tma" -s 2 -c 1 -o gpurun_out/gpu34_k1g_q4 python scripts/k1_timing.py q4 3 > gpurun_out/gpu34_ncu.log 2>&1
