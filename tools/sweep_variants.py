"""Times every FFMA tile variant on every distinct layer of a config (CUDA
events, median of repeats) -- input for the tile selector heuristic."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_10170_b200 import nets  # noqa: E402


def main(config="vgg16", batch=32, reps=5):
    seen = {}
    for l in nets.CONFIGS[config]:
        if l.first:
            continue
        key = (l.c_i, l.c_o, l.h_i, l.w_i, l.h_f, l.s)
        if key in seen:
            continue
        x = nets.Act(batch, l.c_i, l.h_i, l.w_i)
        x.buf.uniform_(-1, 1)
        w = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), device="cuda").uniform_(-1, 1)
        wb = nets.pack_weights(w, False)
        y = nets.Act(batch, l.c_o, l.h_o, l.w_o)
        res = {}
        for v in (1, 2, 3):  # dconv_conv_desc.tile_variant
            ts = []
            for r in range(reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                nets.conv(l, batch, x, wb, y, tile_variant=v)
                b.record()
                b.synchronize()
                if r:
                    ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            res[v] = round(batch * l.flops / (ms * 1e-3) / 1e12, 2)
        seen[key] = res
        print(json.dumps({"layer": l.name, "shape": key, "tflops_by_variant": res}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "vgg16",
         int(sys.argv[2]) if len(sys.argv) > 2 else 32)
