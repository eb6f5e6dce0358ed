set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/gpu36_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu36_pytest.log
timeout 600 python scripts/energy_timing.py weak1 5 > gpurun_out/gpu36_energy.log 2>&1
