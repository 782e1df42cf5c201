"""Split-K factor sweep for the batch-1 layers (cfg1, AlexNet conv2-5,
ResNet-50 b1 stage 3/4 shapes): every CTA tile x forced cluster size ks
(DCONV_KSPLIT, read per launch) against the launcher's own choice; kernel
time by CUDA events over 20 back-to-back launches.
usage: python tools/ks_sweep.py [out.jsonl]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_10170_b200 import nets  # noqa: E402

LAYERS = [nets.CFG1[0]] + nets.ALEXNET[1:] + [
    nets.Layer("r50_s3_3x3", 256, 256, 16, 16, 3, 3, 1),
    nets.Layer("r50_s4_3x3", 512, 512, 9, 9, 3, 3, 1),
    nets.Layer("r50_s3_1x1", 1024, 256, 14, 14, 1, 1, 1)]


def t_us(run, reps=20):
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        a.record()
        for _ in range(reps):
            run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    return statistics.median(ts)


out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
for l in LAYERS:
    x = nets.Act(1, l.c_i, l.h_i, l.w_i)
    x.buf.uniform_(-1, 1)
    w = nets.pack_weights(torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), device="cuda").uniform_(-1, 1),
                          False)
    y = nets.Act(1, l.c_o, l.h_o, l.w_o)
    rec = {"layer": l.name, "gflop": l.flops / 1e9, "auto": {}, "forced": {}}
    for tv in (1, 2, 3):
        os.environ.pop("DCONV_KSPLIT", None)
        rec["auto"][tv] = round(t_us(lambda: nets.conv(l, 1, x, w, y, 1, tile_variant=tv)), 2)
        for ks in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16):
            os.environ["DCONV_KSPLIT"] = str(ks)
            rec["forced"][f"{tv}/{ks}"] = round(t_us(lambda: nets.conv(l, 1, x, w, y, 1,
                                                                       tile_variant=tv)), 2)
        os.environ.pop("DCONV_KSPLIT", None)
    best = min(rec["forced"].items(), key=lambda kv: kv[1])
    rec["best_forced"] = best
    rec["best_auto"] = min(rec["auto"].items(), key=lambda kv: kv[1])
    print(json.dumps({k: rec[k] for k in ("layer", "auto", "best_forced", "best_auto")}), flush=True)
    if out:
        out.write(json.dumps(rec) + "\n")
