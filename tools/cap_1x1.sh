#!/bin/bash
# ncu --set full captures WITH the source page (per-SASS-line warp-state
# samples) of ResNet-50 b256 1x1 layers on the FFMA kernel; the text exports
# come back in gpurun_out/cap1x1 (the .ncu-rep is dropped: gpurun returns
# <= 64 MiB).  Read them with tools/ncu_quick.py-style sums per SASS region;
# profiles/r2_ncu_src_1x1.txt holds what was found.  Run under gpurun:
#   gpurun -- 'bash tools/cap_1x1.sh'
set -u
O=gpurun_out/cap1x1; mkdir -p $O
full() {
  local name=$1 k=$2; shift 2
  python tools/one_layer.py "$@" > $O/plain_$name.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s ${FS:-3} -c 1 \
    -o $O/full_$name python tools/one_layer.py "$@" > $O/ncu_$name.log 2>&1
  ncu -i $O/full_$name.ncu-rep --page raw --csv > $O/full_$name.raw.csv 2>/dev/null
  ncu -i $O/full_$name.ncu-rep --page source --csv > $O/full_$name.src.csv 2>/dev/null
  rm -f $O/full_$name.ncu-rep
}
export DCONV_NO_TAILSPLIT=1
FS=4 full r50_s1c3 conv_ffma 64 256 56 56 1 1 256 3 ffma_add
FS=4 full r50_s3c1 conv_ffma 1024 256 14 14 1 1 256 3 ffma
FS=4 full r50_s3c2 conv_ffma 256 256 16 16 3 1 256 3 ffma
