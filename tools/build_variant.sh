#!/bin/bash
# A/B build of the product library with extra nvcc defines, into build_var/<name>/libsst_gpu.so
# (select it at run time with SST_GPU_LIB=build_var/<name>/libsst_gpu.so).
#   tools/build_variant.sh <name> -DSST_WF_LOGIC_BLOCKS=4 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build_var/$name
mkdir -p $out
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $*"
C=paper_2011_03082_b200/csrc
nvcc $FL -c $C/kernels_f32.cu -o $out/kernels_f32.o &
nvcc $FL -fmad=false -c $C/kernels_f64.cu -o $out/kernels_f64.o &
nvcc $FL -fmad=false -c $C/train.cu -o $out/train.o &
nvcc $FL -c $C/api.cu -o $out/api.o &
nvcc $FL -x cu -c $C/host.cpp -o $out/host.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libsst_gpu.so \
    $out/kernels_f32.o $out/kernels_f64.o $out/train.o $out/api.o $out/host.o
echo "built $out/libsst_gpu.so"
