set -x
nvidia-smi > /dev/null
for w in 4 1 2; do BMV_K1_WPC=$w timeout 600 python scripts/k1_timing.py weak1 10 >> gpurun_out/gpu39_k1.log 2>&1; BMV_K1_WPC=$w timeout 600 python scripts/k1_timing.py q4 10 >> gpurun_out/gpu39_k1.log 2>&1; done
timeout 900 python scripts/om_breakdown.py weak1 > gpurun_out/gpu39_om.log 2>&1
