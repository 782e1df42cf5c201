#!/bin/bash
# Builds paper_1809_10170_b200/libdconv_b200_prof.so: the product library with
# the kernels' clock instrumentation compiled in (-DDCONV_FFMA_PROF,
# -DDCONV_TF32_PROF, -DDCONV_X3_PROF): per-CTA phase clocks / per-role wait
# cycles printed by DCONV_FFMA_PROFILE=1 / DCONV_TF32_PROFILE=1.  Use it with
# DCONV_LIB=...; not for timed runs (the product build has none of it).
set -e
cd "$(dirname "$0")/../paper_1809_10170_b200/csrc"
make -s >/dev/null 2>&1 || true
mkdir -p build_prof
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I."
for f in conv_ffma conv_tf32 conv_tf32x3; do
  $NV -DDCONV_FFMA_PROF -DDCONV_TF32_PROF -DDCONV_X3_PROF -c $f.cu -o build_prof/$f.o &
done
wait
objs=$(ls build/*.o | grep -v -e conv_ffma.o -e conv_tf32.o -e conv_tf32x3.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libdconv_b200_prof.so \
  $objs build_prof/conv_ffma.o build_prof/conv_tf32.o build_prof/conv_tf32x3.o -lcudart
echo built ../libdconv_b200_prof.so
