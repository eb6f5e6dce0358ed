set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x -k "projection or smoke" > gpurun_out/gpu33_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu33_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu33_spmm.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4_lane|k5_lane" -s 2 -c 2 -o gpurun_out/gpu33_lane_proj python scripts/spmm_timing.py proj 3 > gpurun_out/gpu33_ncu.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and slow" -q -k "projection" > gpurun_out/gpu33_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu33_pytest_slow.log
