set -x
nvidia-smi > /dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/gpu29_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu29_pytest.log
for cfg in q4 weak1; do for fz in 1 0; do BMV_K1_FUSED_ZERO=$fz timeout 600 python scripts/apply_timing.py $cfg 10 >> gpurun_out/gpu29_apply.log 2>&1; done; done
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/gpu29_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/gpu29_bench.log
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/gpu29_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu29_pytest_slow.log
