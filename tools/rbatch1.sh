# batch-1 layers (AlexNet, cfg1, ResNet/VGG b1 shapes): split-K cluster choice
cd /root/repo
for shp in "64 64 58 58 3 1 1" "96 256 31 31 5 1 1" "256 384 15 15 3 1 1" "384 384 15 15 3 1 1" "384 256 15 15 3 1 1" "512 512 16 16 3 1 1" "512 512 9 9 3 1 1" "1024 256 14 14 1 1 1" "64 64 226 226 3 1 1"; do
  DCONV_DEBUG=1 python tools/one_layer.py $shp 3 2>&1 | sort | uniq -c | sort -rn | head -3
done
