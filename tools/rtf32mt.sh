# TF32 kernel: channels per unit (N) x M-tiles per unit (MT) sweep on VGG b32 shapes
cd /root/repo
for shp in "128 128 114 114 3 1 32" "256 256 58 58 3 1 32" "512 512 30 30 3 1 32" "512 512 16 16 3 1 32"; do
  for nm in "0 0" "128 1" "128 2" "128 4" "256 1" "256 2"; do
    set -- $nm
    if [ "$1" = "0" ]; then e=""; else e="DCONV_TF32_N=$1 DCONV_TF32_MT=$2"; fi
    echo "N=$1 MT=$2: $(env $e python tools/one_layer.py $shp 3 tf32 | tail -1)"
  done
done
