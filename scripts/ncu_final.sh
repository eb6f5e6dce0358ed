# ncu --set full captures of the shipped kernels (one launch each) per config, summarised on
# the GPU box (the reports are too large to bring back together):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash scripts/ncu_final.sh r02'
TAG=${1:-r02}
mkdir -p gpurun_out /tmp/ncu_final
for cfg in weak1 q4 proj q2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_(plane|pair)_kernel|chunk_kernel' \
    --launch-skip 3 -c 3 -o /tmp/ncu_final/${TAG}_final_${cfg} -f python scripts/prof_k1.py $cfg 2 > gpurun_out/${TAG}_ncu_${cfg}.log 2>&1
  { echo "# ncu --set full, ${cfg}: K1, K4, K5 as shipped (one launch each, --clock-control none)"; echo;
    python scripts/ncu_summary.py /tmp/ncu_final/${TAG}_final_${cfg}.ncu-rep;
    echo; echo "## Instruction mix and hottest source lines"; echo;
    python scripts/ncu_source.py /tmp/ncu_final/${TAG}_final_${cfg}.ncu-rep "" 14; } > gpurun_out/${TAG}_final_${cfg}_ncu_full.md 2>&1
done
python scripts/h2d_bw.py > gpurun_out/${TAG}_h2d_bw.log 2>&1
