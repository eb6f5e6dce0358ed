# Per-kernel timings and bench lines on one B200 (run with gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/measure.sh TAG'
TAG=${1:-m}
mkdir -p gpurun_out
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/k1_timing.py $cfg 20 >> gpurun_out/${TAG}_k1.log 2>&1; done
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 20 >> gpurun_out/${TAG}_spmm.log 2>&1; done
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_weak1.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_bench_weak1.log
for cfg in q2 q4 proj; do timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_bench_cfgs.log 2>&1; done
