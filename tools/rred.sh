# split-K reduction cost constants of the batch-1 cost model
cd /root/repo
for rc in "1500 300" "4000 400" "6000 600"; do
  set -- $rc
  echo "== red0=$1 red1=$2"
  for c in cfg1 alexnet; do
    DCONV_RED0=$1 DCONV_RED1=$2 python bench.py --config $c --no-cpu-baseline --no-tune 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'])"
  done
  DCONV_RED0=$1 DCONV_RED1=$2 python bench.py --config googlenet --batch 1 --no-cpu-baseline --no-tune 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('googlenet b1', d['value'], d['ms_per_step'])"
done
