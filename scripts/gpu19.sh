set -x
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu19_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu19_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu19_spmm.log 2>&1; done
timeout 300 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu19_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pj_stream" -s 1 -c 1 -o gpurun_out/gpu19_pj_q4 python scripts/spmm_timing.py q4 3 > gpurun_out/gpu19_ncu.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pm_stream" -s 1 -c 1 -o gpurun_out/gpu19_pm_q4 python scripts/spmm_timing.py q4 3 >> gpurun_out/gpu19_ncu.log 2>&1
timeout 900 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/gpu19_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu19_pytest_slow.log
