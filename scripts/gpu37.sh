set -x
nvidia-smi > /dev/null
timeout 600 python scripts/spmm_timing.py proj 3 > gpurun_out/gpu37_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4_lane|k5_lane" -s 2 -c 2 -o gpurun_out/gpu37_lane_proj python scripts/spmm_timing.py proj 3 > gpurun_out/gpu37_ncu.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/gpu37_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/gpu37_smoke.log
