#!/bin/bash
# One GPU call that refreshes the round's measured evidence (results land in
# gpurun_out/round; tools/save_round.py + tools/ncu_summary.py turn them into
# profiles/ summaries).
#   1. bench.py default (VGG-16 b32 FFMA headline + every other config as
#      extra_configs + the CPU baseline), the split-TF32 and TF32 paths, the
#      CPU reference arm, C_o-sharded ResNet-50 b1 (NCCL / fused peer, 1 rank)
#   2. ncu launch list of one VGG-16 b32 step (FFMA and split-TF32)
#   3. ncu --set full of the top kernels: FFMA VGG conv1_2 / conv4_2 and two
#      ResNet-50 b256 1x1 layers (64->256 56x56, 256->1024 14x14, skip-add), the
#      TMA-store first-layer reader (VGG conv1_1 b32, 7x7/s2 stem b64),
#      split-TF32 VGG conv4_2 and ResNet 1024->256 1x1
#   (direct vs im2col vs cuDNN: IM2COL=1)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvidia_smi.txt 2>&1
T="timeout 600"

T0=$SECONDS; $T python bench.py > $O/bench_default.log 2>&1; echo "bench default wall $((SECONDS - T0)) s" > $O/bench_default_wall.txt
for a in tf32x3 tf32; do
  $T python bench.py --algo $a --no-cpu-baseline > $O/bench_$a.log 2>&1
done
$T python bench.py --impl reference > $O/bench_reference.log 2>&1
$T python bench.py --config resnet50 --shard co --no-cpu-baseline > $O/bench_resnet50_co_nccl.log 2>&1
$T python bench.py --config resnet50 --shard co --gather peer --no-cpu-baseline > $O/bench_resnet50_co_peer.log 2>&1

# per-rank workloads of the batch-sharded configs at 2 / 4 / 8 ranks (no
# collective on that path: N ranks run N of these side by side), and the
# stream-K / split-tail A/B of the headline
for b in 16 8 4; do $T python bench.py --batch $b --extra none --no-cpu-baseline > $O/scale_vgg16_b$b.log 2>&1; done
for b in 128 64 32; do $T python bench.py --config resnet50 --batch $b --extra none --no-cpu-baseline > $O/scale_resnet50_b$b.log 2>&1; done
for c in vgg16 resnet50; do DCONV_NO_STREAMK=1 $T python bench.py --config $c --extra none --no-cpu-baseline > $O/nostreamk_$c.log 2>&1; done

L="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tune --extra none"
$L > $O/plain_launches.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_vgg16.csv $L > $O/ncu_launches.log 2>&1
$L --algo tf32x3 > $O/plain_launches_x3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_vgg16_tf32x3.csv $L --algo tf32x3 > $O/ncu_launches_x3.log 2>&1

full() {  # name kernel-regex one_layer args...  (FS: launches to skip; tail-split FFMA layers launch twice)
  local name=$1 k=$2; shift 2
  python tools/one_layer.py "$@" > $O/plain_full_$name.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s ${FS:-3} -c 1 \
    -o $O/full_$name python tools/one_layer.py "$@" > $O/ncu_full_$name.log 2>&1
  # text exports only (gpurun brings back <= 64 MiB): raw counters + source page
  ncu -i $O/full_$name.ncu-rep --page raw --csv > $O/full_$name.raw.csv 2>/dev/null
  ncu -i $O/full_$name.ncu-rep --page source --csv > $O/full_$name.src.csv 2>/dev/null
  rm -f $O/full_$name.ncu-rep
}
FS=4 full conv1_2 conv_ffma 64 64 226 226 3 1 32 3
FS=4 full conv4_2 conv_ffma 512 512 30 30 3 1 32 3
FS=4 full ffma_r50_s1c3 conv_ffma 64 256 56 56 1 1 256 3 ffma_add
FS=4 full ffma_r50_s3c3 conv_ffma 256 1024 14 14 1 1 256 3 ffma_add
full reader_conv1_1 conv_reader 3 64 226 226 3 1 32 3 first
full reader_stem conv_reader 3 64 229 229 7 2 64 3 first
full x3_conv4_2 conv_tf32x3 512 512 30 30 3 1 32 3 tf32x3
full x3_r50_1x1 conv_tf32x3 1024 256 14 14 1 1 256 3 tf32x3

if [ -n "${IM2COL:-}" ]; then
  for c in cfg1 alexnet googlenet vgg16 resnet50; do
    python tools/compare_im2col.py --config $c --json $O/im2col_$c.json > $O/im2col_$c.log 2>&1
  done
fi
du -sh $O > $O/du.txt
echo done
