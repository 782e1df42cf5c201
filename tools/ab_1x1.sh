# A/B of the dense 1x1 consumer loop on ResNet-50 b256 1x1 layers
for args in "1024 256 14 14 1 1 256 3 ffma" "256 1024 14 14 1 1 256 3 ffma_add" "256 64 56 56 1 1 256 3 ffma" "64 256 56 56 1 1 256 3 ffma_add" "512 128 28 28 1 1 256 3 ffma" "128 512 28 28 1 1 256 3 ffma_add" "2048 512 7 7 1 1 256 3 ffma" "512 2048 7 7 1 1 256 3 ffma_add"; do
  echo "dense:   $(python tools/one_layer.py $args)"
  echo "general: $(DCONV_NO_DENSE1X1=1 python tools/one_layer.py $args)"
done
