H=$PWD/paper_1809_10170_b200/libdconv_b200_head.so
for args in "64 256 56 56 1 1 256 3 ffma_add" "128 512 28 28 1 1 256 3 ffma_add" "256 1024 14 14 1 1 256 3 ffma_add" "64 64 226 226 3 1 32 3 ffma" "512 512 16 16 3 1 32 3 ffma"; do
  echo "new:  $(python tools/one_layer.py $args)"
  echo "head: $(DCONV_LIB=$H python tools/one_layer.py $args)"
  echo "new:  $(python tools/one_layer.py $args)"
  echo "head: $(DCONV_LIB=$H python tools/one_layer.py $args)"
done
for c in resnet50; do
for i in 1 2; do
python bench.py --config $c --extra none --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('new', d[\"value\"], d[\"ms_per_step\"], d[\"roofline\"][\"frac\"])"
DCONV_LIB=$H python bench.py --config $c --extra none --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('head', d[\"value\"], d[\"ms_per_step\"], d[\"roofline\"][\"frac\"])"
done; done
