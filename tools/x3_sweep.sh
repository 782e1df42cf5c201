#!/bin/bash
# N / MT sweep of the split-TF32 kernel on ResNet-50 / VGG layer shapes (one
# process per setting: the knobs are read once).  Results: gpurun_out/x3sweep.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/x3sweep.txt; : > $O
run() { echo "N=$1 MT=$2 $3: $(DCONV_TF32_N=$1 DCONV_TF32_MT=$2 timeout 60 python tools/one_layer.py $3 2>&1 | tail -1)" >> $O; }
for shape in "64 256 56 56 1 1 256 3 tf32x3_add" "256 64 56 56 1 1 256 3 tf32x3" "1024 256 14 14 1 1 256 3 tf32x3" \
             "256 1024 14 14 1 1 256 3 tf32x3_add" "512 128 28 28 1 1 256 3 tf32x3" "128 512 28 28 1 1 256 3 tf32x3_add" \
             "2048 512 7 7 1 1 256 3 tf32x3" "512 2048 7 7 1 1 256 3 tf32x3_add" \
             "256 256 16 16 3 1 256 3 tf32x3" "512 512 9 9 3 1 256 3 tf32x3" "64 64 58 58 3 1 256 3 tf32x3" \
             "128 128 30 30 3 1 256 3 tf32x3" "512 512 30 30 3 1 32 3 tf32x3" "256 256 58 58 3 1 32 3 tf32x3"; do
  for nm in "256 1" "128 1" "128 2" "64 2" "64 4"; do run $nm "$shape"; done
done
