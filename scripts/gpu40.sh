set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gpu40_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu40_pytest.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu40_spmm.log 2>&1; done
timeout 900 python scripts/om_breakdown.py weak1 > gpurun_out/gpu40_om.log 2>&1
timeout 600 python scripts/energy_timing.py weak1 5 > gpurun_out/gpu40_energy.log 2>&1
