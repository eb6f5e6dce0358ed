set -x
nvidia-smi > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_peaks.cu -o /tmp/fp64_peaks && /tmp/fp64_peaks > gpurun_out/gpu22_peaks.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu22_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu22_pytest.log
for cfg in q2 q4 weak1; do
  for v in "stream 1" "stream 0" "onepass 1"; do
    set -- $v
    BMV_K1=$1 BMV_K1_XPF=$2 timeout 600 python scripts/k1_timing.py $cfg 10 >> gpurun_out/gpu22_k1.log 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cellop_stream" -s 2 -c 1 -o gpurun_out/gpu22_k1s_q4 python scripts/k1_timing.py q4 3 > gpurun_out/gpu22_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pj_stream|pm_stream" -s 2 -c 2 -o gpurun_out/gpu22_spmm_w1 python scripts/spmm_timing.py weak1 3 >> gpurun_out/gpu22_ncu.log 2>&1
timeout 900 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/gpu22_pytest_slow.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu22_pytest_slow.log
