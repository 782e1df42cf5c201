"""Runs chosen launches of a config's plan (autotuned tiles, as the bench runs
them) a few times: for ncu captures of one layer in its real context.
usage: python tools/plan_layer.py CONFIG BATCH NAME[,NAME...] [reps] [algo]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_10170_b200 import nets  # noqa: E402

config, n, names = sys.argv[1], int(sys.argv[2]), sys.argv[3].split(",")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
algo = sys.argv[5] if len(sys.argv) > 5 else "ffma"
plan = nets.build_plan(config, n, algo=algo)
tiles = plan.autotune()
plan.run()
steps = [s for s in plan.steps if s.name in names]
assert steps, [s.name for s in plan.steps]
torch.cuda.synchronize()
for s in steps:
    torch.cuda.nvtx.range_push("target")  # ncu --nvtx --nvtx-include "target/"
    for _ in range(reps):
        s.fn(None)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        s.fn(None)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"{s.name} tile {tiles.get(s.name)}: {ms * 1e3:.1f} us, "
          f"{s.flops / ms / 1e9:.1f} TFLOP/s", flush=True)
