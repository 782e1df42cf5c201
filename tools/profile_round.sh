#!/bin/bash
# One GPU call that refreshes the round's measured evidence (results land in
# gpurun_out/round; tools/save_round.py + tools/ncu_summary.py turn them into
# profiles/ summaries).
#   1. bench.py, every config: FFMA (headline), TF32, split-TF32 (x3), + the CPU arm
#   2. ncu launch lists of the default bench command and of VGG-16 b32 tf32x3
#   3. ncu --set full of the top kernels (FFMA: VGG conv1_2 / conv4_2;
#      tf32x3: VGG conv4_2, ResNet 1024->256 1x1)
#   4. C_o-sharded ResNet-50 b1, NCCL and fused peer gather (1 rank)
#   (direct vs im2col vs cuDNN: IM2COL=1)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvidia_smi.txt 2>&1
T="timeout 300"

T0=$SECONDS; $T python bench.py > $O/bench_vgg16_ffma.log 2>&1; echo "bench default wall $((SECONDS - T0)) s" > $O/bench_default_wall.txt
for c in resnet50 googlenet alexnet cfg1; do
  $T python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_ffma.log 2>&1
done
for a in tf32 tf32x3; do
  for c in vgg16 resnet50 googlenet alexnet cfg1; do
    $T python bench.py --config $c --algo $a --no-cpu-baseline > $O/bench_${c}_$a.log 2>&1
  done
done
$T python bench.py --impl reference > $O/bench_reference.log 2>&1
$T python bench.py --config resnet50 --shard co --no-cpu-baseline > $O/bench_resnet50_co_nccl.log 2>&1
$T python bench.py --config resnet50 --shard co --gather peer --no-cpu-baseline > $O/bench_resnet50_co_peer.log 2>&1

timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_vgg16.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $O/ncu_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_vgg16_tf32x3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --algo tf32x3 > $O/ncu_launches_x3.log 2>&1

full() {  # name kernel-regex one_layer args...
  local name=$1 k=$2; shift 2
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o $O/full_$name python tools/one_layer.py "$@" > $O/ncu_full_$name.log 2>&1
}
full conv1_2 conv_ffma 64 64 226 226 3 1 32 1
full conv4_2 conv_ffma 512 512 30 30 3 1 32 1
full x3_conv4_2 conv_tf32x3 512 512 30 30 3 1 32 1 tf32x3
full x3_r50_1x1 conv_tf32x3 1024 256 14 14 1 1 256 1 tf32x3

if [ -n "${IM2COL:-}" ]; then
  for c in cfg1 alexnet googlenet vgg16 resnet50; do
    python tools/compare_im2col.py --config $c --json $O/im2col_$c.json > $O/im2col_$c.log 2>&1
  done
fi
echo done
