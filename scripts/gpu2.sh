set -x
timeout 900 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu2_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu2_pytest.log
timeout 600 python bench.py --config q2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gpu2_bench_q2.log 2>&1
timeout 600 python bench.py --config q4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gpu2_bench_q4.log 2>&1
timeout 300 python scripts/prof_k1.py q2 3 > gpurun_out/gpu2_plain_q2.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gpu2_launches_q2.csv python scripts/prof_k1.py q2 3 > gpurun_out/gpu2_ncu_launch.log 2>&1
timeout 300 python scripts/prof_k1.py q4 2 > gpurun_out/gpu2_plain_q4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cellop_kernel -s 1 -c 1 -o gpurun_out/gpu2_k1_q4 python scripts/prof_k1.py q4 2 > gpurun_out/gpu2_ncu_full.log 2>&1
timeout 300 python scripts/prof_k1.py q2 2 > gpurun_out/gpu2_plain_q2b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tm_partial|mmult_kernel|cellop_kernel" -s 3 -c 3 -o gpurun_out/gpu2_q2_kernels python scripts/prof_k1.py q2 2 > gpurun_out/gpu2_ncu_full2.log 2>&1
