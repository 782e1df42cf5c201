H=$PWD/paper_1809_10170_b200/libdconv_b200_head.so
for a in tf32x3 tf32; do for c in resnet50 vgg16 googlenet; do
python bench.py --config $c --algo $a --extra none --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('new $a $c', d[\"value\"], d[\"ms_per_step\"])"
DCONV_LIB=$H python bench.py --config $c --algo $a --extra none --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('head $a $c', d[\"value\"], d[\"ms_per_step\"])"
done; done
