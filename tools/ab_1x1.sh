# A/B of 256-bit pencil loads / stores in the FFMA epilogues (DCONV_NO_WIDE_IO=1: two 128-bit halves)
for args in "64 256 56 56 1 1 256 3 ffma_add" "128 512 28 28 1 1 256 3 ffma_add" "256 1024 14 14 1 1 256 3 ffma_add" "512 2048 7 7 1 1 256 3 ffma_add" "256 64 56 56 1 1 256 3 ffma" "64 64 226 226 3 1 32 3 ffma" "64 64 58 58 3 1 1 3 ffma"; do
  echo "256-bit: $(python tools/one_layer.py $args)"
  echo "128-bit: $(DCONV_NO_WIDE_IO=1 python tools/one_layer.py $args)"
done
