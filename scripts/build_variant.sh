# Build an experimental libbmv variant: bash scripts/build_variant.sh NAME [nvcc flags...]
# -> scripts/tmp/libbmv_NAME.so (use with BMV_LIB=scripts/tmp/libbmv_NAME.so)
NAME=$1; shift
mkdir -p scripts/tmp
C=paper_1907_01005_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  -I include -I $C "$@" $C/bmv_util.cu $C/bmv_misc.cu $C/bmv_k1.cu $C/bmv_spmm.cu -o scripts/tmp/libbmv_$NAME.so
