"""Accuracy probe: split-TF32 with the main term accumulated in K chunks.

Like tools/tf32x3_accuracy.py, but T(x_hi, w_hi) runs over input-channel
chunks of `cc` channels (K chunk = cc * H_f * W_f) and the chunk results are
summed in fp32 (what a kernel that drains a TMEM accumulator into registers
every chunk would do); the two correction terms run over the full K.
Tool only (uses oracle/ as the checker).
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from oracle import pyoracle as po  # noqa: E402
from tf32x3_accuracy import report, split, tf32_conv  # noqa: E402


def main():
    cases = [(256, 256, 16, 16, 3, 2), (512, 512, 30, 30, 3, 1), (512, 512, 9, 9, 3, 2),
             (2048, 512, 9, 9, 1, 2)]
    for ci, co, h, w, f, n in cases:
        x = po.uniform((n, ci, h, w), 4242 + ci, co)
        k = po.uniform((ci, co, f, f), 4343 + ci, co)
        want = np.stack([po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8) for i in range(n)])
        print(f"{ci}->{co} {h}x{w} f{f} n{n} (K={ci * f * f})", flush=True)
        xh, xl = split(x, "trunc")
        kh, kl = split(k, "trunc")
        corr = tf32_conv(xh, kl) + tf32_conv(xl, kh)
        for cc in (8, 16, 32, 64, 128):
            if cc >= ci:
                continue
            main_t = np.zeros_like(corr)
            for c0 in range(0, ci, cc):
                main_t = (main_t + tf32_conv(np.ascontiguousarray(xh[:, c0:c0 + cc]),
                                             np.ascontiguousarray(kh[c0:c0 + cc]))).astype(np.float32)
            report(f"cc{cc} K{cc * f * f}", (main_t + corr).astype(np.float32), want)
            # corrections chunked too (all three terms into one chunk accumulator)
            tot = np.zeros_like(corr)
            for c0 in range(0, ci, cc):
                sl = slice(c0, c0 + cc)
                a, b = np.ascontiguousarray(xh[:, sl]), np.ascontiguousarray(kh[sl])
                t = tf32_conv(a, b) + tf32_conv(a, np.ascontiguousarray(kl[sl])) + \
                    tf32_conv(np.ascontiguousarray(xl[:, sl]), b)
                tot = (tot + t).astype(np.float32)
            report(f"  all3 cc{cc}", tot, want)


if __name__ == "__main__":
    main()
