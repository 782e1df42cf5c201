#!/bin/bash
# One GPU call that refreshes the round's measured evidence (results land in
# gpurun_out/; tools/ncu_summary.py turns them into profiles/ summaries).
#   1. bench.py, every config, FFMA (headline) and TF32 variant, + the CPU arm
#   2. ncu launch list of the default bench command (per-launch durations)
#   3. ncu --set full of the top conv kernels (VGG conv1_2, conv4_2 at b32)
#   4. direct vs im2col+SGEMM vs cuDNN on every config
#   5. C_o-sharded ResNet-50 b1, NCCL and fused peer gather (1 rank)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvidia_smi.txt 2>&1

T0=$SECONDS; python bench.py > $O/bench_vgg16_ffma.log 2>&1; echo "bench default wall $((SECONDS - T0)) s" > $O/bench_default_wall.txt
for c in resnet50 googlenet alexnet cfg1; do
  python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_ffma.log 2>&1
done
for c in vgg16 resnet50 googlenet alexnet cfg1; do
  python bench.py --config $c --algo tf32 --no-cpu-baseline > $O/bench_${c}_tf32.log 2>&1
done
python bench.py --impl reference > $O/bench_reference.log 2>&1
python bench.py --config resnet50 --shard co --no-cpu-baseline > $O/bench_resnet50_co_nccl.log 2>&1
python bench.py --config resnet50 --shard co --gather peer --no-cpu-baseline > $O/bench_resnet50_co_peer.log 2>&1

timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_vgg16.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $O/ncu_launches.log 2>&1

timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_ffma -c 1 \
  -o $O/full_conv1_2 python tools/one_layer.py 64 64 226 226 3 1 32 1 > $O/ncu_full1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_ffma -c 1 \
  -o $O/full_conv4_2 python tools/one_layer.py 512 512 30 30 3 1 32 1 > $O/ncu_full4.log 2>&1

for c in cfg1 alexnet googlenet vgg16 resnet50; do
  python tools/compare_im2col.py --config $c --json $O/im2col_$c.json > $O/im2col_$c.log 2>&1
done
echo done
