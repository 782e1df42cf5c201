set -u
O=gpurun_out/s5b; mkdir -p $O
full() {
  local name=$1 k=$2; shift 2
  python tools/one_layer.py "$@" > $O/plain_$name.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s ${FS:-3} -c 1 \
    -o $O/full_$name python tools/one_layer.py "$@" > $O/ncu_$name.log 2>&1
  ncu -i $O/full_$name.ncu-rep --page raw --csv > $O/full_$name.raw.csv 2>/dev/null
  ncu -i $O/full_$name.ncu-rep --page source --csv > $O/full_$name.src.csv 2>/dev/null
  rm -f $O/full_$name.ncu-rep
}
FS=4 full r50_s3c1 conv_ffma 1024 256 14 14 1 1 256 3 ffma
FS=4 full r50_s3c3 conv_ffma 256 1024 14 14 1 1 256 3 ffma_add
FS=4 full r50_s3c2 conv_ffma 256 256 16 16 3 1 256 3 ffma
for g in 3 5 6 8; do echo G=$g; DCONV_FORCE_G=$g python tools/one_layer.py 1024 256 14 14 1 1 256 3 ffma; done
echo noepi; DCONV_NO_EPI_WG=1 python tools/one_layer.py 1024 256 14 14 1 1 256 3 ffma
for b in 16 24 32 48; do echo PB=$b; DCONV_PATCH_BUDGET=$b python tools/one_layer.py 1024 256 14 14 1 1 256 3 ffma; done
DCONV_DEBUG=1 python tools/one_layer.py 1024 256 14 14 1 1 256 1 ffma 2>&1 | tail -3
