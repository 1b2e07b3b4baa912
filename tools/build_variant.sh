#!/bin/bash
# Build a tuning variant of libmotif_b200.so with extra nvcc defines:
#   tools/build_variant.sh NAME -DMB_TRI_MINB=2 ...
# -> build_variants/libmotif_b200_NAME.so (load with MB_LIB_PATH=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_1602_04478_b200
out=build_variants/$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ccbin /usr/bin/g++ -Xptxas -v --expt-relaxed-constexpr"
$NV "$@" -c $P/csrc/engine/engine.cu -o $out/engine.o 2> $out/ptxas.log || (cat $out/ptxas.log; exit 1)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o build_variants/libmotif_b200_$name.so \
  $P/build/host/graph.o $P/build/host/plan.o $P/build/host/estimate.o $P/build/capi.o $out/engine.o -lpthread
grep -A2 "tri_hist_kernel" $out/ptxas.log | grep -E "registers|spill" || true
