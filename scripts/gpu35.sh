set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/gpu35_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu35_pytest.log
for cfg in q2 q4 weak1; do timeout 600 python scripts/hm_timing.py $cfg 10 >> gpurun_out/gpu35_hm.log 2>&1; done
timeout 300 python scripts/h2d_bw.py > gpurun_out/gpu35_h2d.log 2>&1
