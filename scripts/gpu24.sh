set -x
nvidia-smi > /dev/null
timeout 300 python scripts/debug_lane.py smoke > gpurun_out/gpu24_dbg.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python scripts/debug_lane.py smoke > gpurun_out/gpu24_memcheck.log 2>&1
timeout 300 compute-sanitizer --tool racecheck --racecheck-report analysis python scripts/debug_lane.py smoke > gpurun_out/gpu24_racecheck.log 2>&1
timeout 300 python scripts/debug_lane.py q2 >> gpurun_out/gpu24_dbg.log 2>&1
