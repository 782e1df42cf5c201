"""Accuracy of the split-TF32 kernel itself (conv_tf32x3_kernel, with the
accumulator chunk of DCONV_X3_CHUNK_K) against the fp64 oracle, next to the
FFMA kernel: max |a-b| / (1e-4 + 1e-5|b|) per case (> 1 fails the fp32 bar).
Tool only (uses oracle/ as the checker).
usage: DCONV_X3_CHUNK_K=288 python tools/x3_kernel_accuracy.py [positive]
("positive": |x|, |w| -- no cancellation, the accumulator grows linearly)"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from oracle import pyoracle as po  # noqa: E402
from tf32x3_accuracy import ffma_conv  # noqa: E402
from paper_1809_10170_b200 import nets  # noqa: E402
import torch  # noqa: E402


def x3_conv(x, k):
    n, ci, hi, wi = x.shape
    _, co, hf, wf = k.shape
    l = nets.Layer("a", ci, co, hi, wi, hf, wf, 1)
    a = nets.Act(n, ci, hi, wi)
    a.buf.copy_(torch.from_numpy(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    wp = nets.prepare_tf32(l, nets.pack_weights(torch.from_numpy(k).cuda(), False), x3=True)
    y = nets.Act(n, co, l.h_o, l.w_o)
    nets.conv_tf32(l, n, a, wp, y, x3=True)
    torch.cuda.synchronize()
    return y.buf.cpu().numpy()


def ratio(got, want):
    err = np.abs(got.astype(np.float64) - want)
    return float((err / (1e-4 + 1e-5 * np.abs(want))).max())


def main():
    pos = len(sys.argv) > 1 and sys.argv[1] == "positive"
    print(f"DCONV_X3_CHUNK_K={os.environ.get('DCONV_X3_CHUNK_K', '144 (default)')}"
          f"{' positive data' if pos else ''}")
    for ci, co, h, w, f, n in [(512, 512, 30, 30, 3, 1), (512, 512, 9, 9, 3, 2),
                               (256, 256, 16, 16, 3, 2), (1024, 256, 14, 14, 1, 2),
                               (2048, 512, 7, 7, 1, 2), (64, 64, 58, 58, 3, 1)]:
        x = po.uniform((n, ci, h, w), 4242 + ci, co)
        k = po.uniform((ci, co, f, f), 4343 + ci, co)
        if pos:
            x, k = np.abs(x), np.abs(k)
        want = np.stack([po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8) for i in range(n)])
        print(f"  {ci}->{co} {h}x{w} f{f} n{n} K={ci * f * f}: err/tol tf32x3 "
              f"{ratio(x3_conv(x, k), want):.3f}  ffma {ratio(ffma_conv(x, k), want):.3f}",
              flush=True)


if __name__ == "__main__":
    main()
