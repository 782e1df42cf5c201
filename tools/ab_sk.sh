# A/B of stream-K (DCONV_NO_STREAMK=1: main waves + split-K tail launch, as before)
for args in "512 512 16 16 3 1 32 3 ffma" "512 512 30 30 3 1 32 3 ffma" "256 256 58 58 3 1 32 3 ffma" "128 128 114 114 3 1 32 3 ffma" "512 512 9 9 3 1 256 3 ffma" "256 256 16 16 3 1 256 3 ffma" "1024 256 14 14 1 1 256 3 ffma" "256 1024 14 14 1 1 256 3 ffma_add" "2048 512 7 7 1 1 256 3 ffma" "512 2048 7 7 1 1 256 3 ffma_add" "96 128 30 30 3 1 64 3 ffma" "112 224 16 16 3 1 64 3 ffma" "512 512 30 30 3 1 4 3 ffma" "256 256 58 58 3 1 4 3 ffma"; do
  echo "stream-K: $(timeout 60 python tools/one_layer.py $args)"
  echo "tail:     $(DCONV_NO_STREAMK=1 timeout 60 python tools/one_layer.py $args)"
done
