#!/bin/bash
# Builds paper_1809_10170_b200/libdconv_b200_x3prof.so: the product library with
# conv_tf32x3.cu compiled with -DDCONV_X3_PROF (per-role wait cycles printed by
# DCONV_TF32_PROFILE=1).  Use it with DCONV_LIB=...; not for timed runs.
set -e
cd "$(dirname "$0")/../paper_1809_10170_b200/csrc"
make -s build/abi.o >/dev/null 2>&1 || true
mkdir -p build_prof
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I."
$NV -DDCONV_X3_PROF -c conv_tf32x3.cu -o build_prof/conv_tf32x3.o
objs=$(ls build/*.o | grep -v conv_tf32x3.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libdconv_b200_x3prof.so $objs build_prof/conv_tf32x3.o -lcudart
echo built ../libdconv_b200_x3prof.so
