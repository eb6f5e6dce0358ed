# K4 / K5 kernel-shape sweep (tuning): bash scripts/spmm_sweep.sh TAG [configs...]
# variants built with scripts/build_variant.sh wWbB -DBMV_SPMM_WARPS=W -DBMV_SPMM_BUFS=B
TAG=${1:-sweep}; shift
CFGS=${@:-"proj weak1"}
for lib in default $(ls scripts/tmp | grep '^libbmv_w' | sed 's/libbmv_//; s/.so//'); do
  for cfg in $CFGS; do
    L=""; [ $lib != default ] && L=scripts/tmp/libbmv_$lib.so
    echo -n "lib $lib " >> gpurun_out/${TAG}.log
    BMV_LIB=$L timeout 600 python scripts/spmm_timing.py $cfg 20 >> gpurun_out/${TAG}.log 2>&1
  done
done
