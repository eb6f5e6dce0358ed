set -x
nvidia-smi > /dev/null
for cfg in q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 10 >> gpurun_out/gpu41_spmm.log 2>&1; done
timeout 300 python scripts/zero_bw.py > gpurun_out/gpu41_zero.log 2>&1
