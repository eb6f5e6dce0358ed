set -x
nvidia-smi > /dev/null
timeout 300 python scripts/debug_lane.py smoke > gpurun_out/gpu25_dbg.log 2>&1
timeout 300 python scripts/debug_lane.py q2 >> gpurun_out/gpu25_dbg.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gpu25_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu25_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu25_spmm.log 2>&1; done
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/gpu25_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/gpu25_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4_lane|k5_lane" -s 2 -c 2 -o gpurun_out/gpu25_lane_w1 python scripts/spmm_timing.py weak1 3 > gpurun_out/gpu25_ncu.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/gpu25_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu25_pytest_slow.log
