set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/gpu28_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu28_pytest.log
for cfg in q2 q4 weak1; do BMV_K1=tma timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu28_k1.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_tma" -s 2 -c 1 -o gpurun_out/gpu28_k1t_q4 python scripts/k1_timing.py q4 3 > gpurun_out/gpu28_ncu.log 2>&1
timeout 1200 python bench.py > gpurun_out/gpu28_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/gpu28_bench.log
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/gpu28_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu28_pytest_slow.log
