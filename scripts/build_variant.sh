#!/bin/bash
# Build the engine with extra nvcc flags into variants/<name>.so (A/B timing
# with GP_ENGINE_LIB=variants/<name>.so).  Usage: build_variant.sh name -DX=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2505_15536_b200/csrc"
mkdir -p ../../variants
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr"
nvcc $F "$@" -c -o /tmp/v_$name.o engine.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../variants/$name.so /tmp/v_$name.o verify.o
echo built variants/$name.so
