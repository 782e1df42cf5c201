# A/B of the epilogue warpgroup's L2 skip prefetch on ResNet-50 b256 1x1 + skip layers
for args in "64 256 56 56 1 1 256 3 ffma_add" "128 512 28 28 1 1 256 3 ffma_add" "256 1024 14 14 1 1 256 3 ffma_add" "512 2048 7 7 1 1 256 3 ffma_add" "256 64 56 56 1 1 256 3 ffma" "1024 256 14 14 1 1 256 3 ffma"; do
  echo "prefetch:    $(python tools/one_layer.py $args)"
  echo "no prefetch: $(DCONV_NO_EPI_PREFETCH=1 python tools/one_layer.py $args)"
done
