"""Runs one conv layer a few times (for ncu / compute-sanitizer captures).
usage: python tools/one_layer.py CI CO HI WI F S N [reps] [ffma|tf32|tf32x3|first|ffma_add|tf32_add|tf32x3_add]
(first: the first-layer reader on a dense [N][CI][HI][WI] input)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_10170_b200 import nets  # noqa: E402

ci, co, hi, wi, f, s, n = (int(v) for v in sys.argv[1:8])
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 3
algo = sys.argv[9] if len(sys.argv) > 9 else "ffma"
l = nets.Layer("one", ci, co, hi, wi, f, f, s, algo == "first")
if algo == "first":
    x = torch.empty((n, ci, hi, wi), device="cuda").uniform_(-1, 1)
else:
    x = nets.Act(n, ci, hi, wi)
    x.buf.uniform_(-1, 1)
w = nets.pack_weights(torch.empty((ci, co, f, f), device="cuda").uniform_(-1, 1), l.first)
y = nets.Act(n, co, l.h_o, l.w_o)
sk = None
epi = 0
if algo.endswith("_add"):  # ResNet block tail: relu(conv + skip)
    sk = nets.Act(n, co, l.h_o, l.w_o)
    sk.buf.uniform_(-1, 1)
    epi = 3
    algo = algo[:-4]
if algo in ("tf32", "tf32x3"):
    x3 = algo == "tf32x3"
    wp = nets.prepare_tf32(l, w, x3=x3)
    run = lambda: nets.conv_tf32(l, n, x, wp, y, epi, sk, x3=x3)  # noqa: E731
else:
    import os
    tv = int(os.environ.get("TILE", "0"))  # desc.tile_variant (0 = selector)
    run = lambda: nets.conv(l, n, x, w, y, epi, sk, tile_variant=tv)  # noqa: E731
for _ in range(reps):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    run()
b.record()
b.synchronize()
ms = a.elapsed_time(b) / 10
print(f"{algo} layer {ci}->{co} {hi}x{wi} f{f} s{s} n{n}: {ms*1e3:.1f} us, {n*l.flops/ms/1e9:.1f} TFLOP/s")
