set -x
nvidia-smi > /dev/null
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu42_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu42_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/gpu42_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/gpu42_smoke.log
for cfg in q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu42_spmm.log 2>&1; done
timeout 300 python scripts/zero_bw.py > gpurun_out/gpu42_zero.log 2>&1
timeout 1200 python bench.py > gpurun_out/gpu42_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/gpu42_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/gpu42_bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/gpu42_bench_ref.log
