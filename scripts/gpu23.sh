set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -k "projection or smoke" > gpurun_out/gpu23_pytest_spmm.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu23_pytest_spmm.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gpu23_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu23_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu23_spmm.log 2>&1; BMV_DETERMINISTIC=1 timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu23_spmm.log 2>&1; done
for cfg in q4 weak1; do BMV_K1=stream BMV_K1_XPF=0 timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu23_k1.log 2>&1; BMV_K1=stream BMV_K1_XPF=1 timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu23_k1.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4_lane|k5_lane" -s 2 -c 2 -o gpurun_out/gpu23_lane_w1 python scripts/spmm_timing.py weak1 3 > gpurun_out/gpu23_ncu.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/gpu23_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu23_pytest_slow.log
