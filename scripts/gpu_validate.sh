# Full validation on one B200 (run with gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash scripts/gpu_validate.sh TAG'
TAG=${1:-validate}
set -x
mkdir -p gpurun_out
nvidia-smi > /dev/null
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/k1_timing.py $cfg 20 >> gpurun_out/${TAG}_k1.log 2>&1; done
for cfg in q2 q4 proj weak1; do timeout 600 python scripts/spmm_timing.py $cfg 20 >> gpurun_out/${TAG}_spmm.log 2>&1; done
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/${TAG}_bench_ref.log
for cfg in q2 q4 proj; do timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_bench_cfgs.log 2>&1; done
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_bench_short.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
