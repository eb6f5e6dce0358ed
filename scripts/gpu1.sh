set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu1_info.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/gpu1_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/gpu1_smoke.log
timeout 600 python bench.py --config q2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gpu1_bench_q2.log 2>&1
timeout 600 python bench.py --config q4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gpu1_bench_q4.log 2>&1
BMV_SCATTER=color timeout 600 python bench.py --config q4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/gpu1_bench_q4_color.log 2>&1
timeout 900 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/gpu1_pytest_slow.log 2>&1; echo "rc $?" >> gpurun_out/gpu1_pytest_slow.log
