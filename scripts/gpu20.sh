set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu20_smi.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu20_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu20_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/gpu20_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/gpu20_smoke.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu20_spmm.log 2>&1; done
timeout 1200 python bench.py > gpurun_out/gpu20_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/gpu20_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/gpu20_bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/gpu20_bench_ref.log
timeout 900 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/gpu20_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu20_pytest_slow.log
