# TF32 kernel on the VGG-16 b32 layer shapes
cd /root/repo
for shp in "64 64 226 226 3 1 32" "64 128 114 114 3 1 32" "128 128 114 114 3 1 32" "128 256 58 58 3 1 32" "256 256 58 58 3 1 32" "256 512 30 30 3 1 32" "512 512 30 30 3 1 32" "512 512 16 16 3 1 32"; do
  python tools/one_layer.py $shp 3 tf32
done
