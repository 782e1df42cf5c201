# VGG conv5 (14x14 maps, 1.3 waves) and other tail-heavy shapes: tail-split cluster sizes
cd /root/repo
for env in "DCONV_TAIL_POW2=1" "X=1"; do
  for shp in "512 512 16 16 3 1 32" "256 256 16 16 3 1 256" "512 512 9 9 3 1 256" "512 512 30 30 3 1 32"; do
    env $env DCONV_DEBUG=1 python tools/one_layer.py $shp 2 2>&1 | sort | uniq -c | sort -rn | head -12
  done
done
