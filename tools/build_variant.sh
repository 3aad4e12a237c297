#!/bin/bash
# Build a variant of libhelmtg_b200.so with extra nvcc defines into exp/<name>.so
#   tools/build_variant.sh NAME -DFOO=1 ...   (select it at run time with HTG_LIB=exp/NAME.so)
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2509_17494_b200/csrc
OUT=$ROOT/exp/build_$NAME  # object files stay here (.gpurunignore); only exp/$NAME.so travels
mkdir -p $OUT
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-fcx-limited-range,-ffp-contract=off,-march=x86-64-v3 -I$SRC -I$ROOT/include --expt-relaxed-constexpr $*"
pids=()
for f in capi.cu k_fine.cu k_dd.cu k_fdm.cu k_band.cu coarse.cu; do nvcc $FL -c $SRC/$f -o $OUT/${f%.*}.o & pids+=($!); done
for f in setup.cpp fdm.cpp coarse_nd.cpp tri.cpp; do nvcc $FL -x cu -c $SRC/$f -o $OUT/${f%.*}.o & pids+=($!); done
for p in ${pids[@]}; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/exp/$NAME.so $OUT/*.o -lcudart
echo built exp/$NAME.so
