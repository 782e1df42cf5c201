"""Accuracy probe for a split-TF32 ("3xTF32") scheme on the tcgen05 kernel.

x = x_hi + x_lo, w = w_hi + w_lo with x_hi = tf32(x); then
conv(x, w) ~= T(x_hi, w_hi) + T(x_hi, w_lo) + T(x_lo, w_hi), each T a TF32
tensor-core conv with fp32 accumulation (the existing dconv_cuda_conv_direct_tf32
kernel, three launches, summed in fp32 here).  Compared against the fp64
oracle with the fp32 tolerance |a-b| <= 1e-4 + 1e-5|b|, next to the FFMA
kernel's error on the same inputs.  Tool only (uses oracle/ as the checker).
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pyoracle as po  # noqa: E402
from paper_1809_10170_b200 import _abi, nets  # noqa: E402
from paper_1809_10170_b200 import dconv as D  # noqa: E402


def split(a, mode):
    u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    if mode == "rne":
        u = u + 0xFFF + ((u >> 13) & 1)
    hi = (u & 0xFFFFE000).astype(np.uint32).view(np.float32)
    return hi, (a.astype(np.float32) - hi).astype(np.float32)


def tf32_conv(xs, k):
    n, ci, hi, wi = xs.shape
    _, co, hf, wf = k.shape
    shape = D.ConvShape(ci, co, hi, wi, hf, wf, 1)
    d = D.make_desc(shape, n, 8, 8, 0)
    xb = torch.from_numpy(np.stack([po.pack_feature_map(xs[i], 8) for i in range(n)])).cuda()
    kb = torch.from_numpy(po.pack_kernel(k, 8, 8)).cuda()
    sz = ctypes.c_int64(0)
    _abi.check(_abi.lib().dconv_cuda_tf32_prepared_size(ctypes.byref(d), ctypes.byref(sz)))
    wp = torch.empty(sz.value, device="cuda")
    _abi.check(_abi.lib().dconv_cuda_prepare_tf32_weights(ctypes.byref(d), _abi.ptr(kb), _abi.ptr(wp),
                                                          _abi.stream_ptr()))
    out = torch.empty((n, (co + 7) // 8, shape.h_o, shape.w_o, 8), device="cuda")
    _abi.check(_abi.lib().dconv_cuda_conv_direct_tf32(ctypes.byref(d), _abi.ptr(xb), _abi.ptr(wp), 0,
                                                      _abi.ptr(out), _abi.stream_ptr()))
    torch.cuda.synchronize()
    return out.cpu().numpy()


def ffma_conv(xs, k):
    n, ci, hi, wi = xs.shape
    _, co, hf, wf = k.shape
    l = nets.Layer("p", ci, co, hi, wi, hf, wf, 1)
    a = nets.Act(n, ci, hi, wi)
    a.buf.copy_(torch.from_numpy(np.stack([po.pack_feature_map(xs[i], 8) for i in range(n)])))
    y = nets.Act(n, co, l.h_o, l.w_o)
    nets.conv(l, n, a, nets.pack_weights(torch.from_numpy(k).cuda(), False), y)
    torch.cuda.synchronize()
    return y.buf.cpu().numpy()


def report(tag, got, want):
    err = np.abs(got.astype(np.float64) - want)
    bound = 1e-4 + 1e-5 * np.abs(want)
    print(f"  {tag:10s} max_abs_err {err.max():.3e}  max err/tol {(err / bound).max():.3f}  "
          f"violations {(err > bound).sum()}", flush=True)


def main():
    cases = [(64, 64, 58, 58, 3, 2), (256, 256, 16, 16, 3, 2), (512, 512, 30, 30, 3, 1),
             (1024, 256, 14, 14, 1, 2), (512, 512, 9, 9, 3, 2)]
    for ci, co, h, w, f, n in cases:
        x = po.uniform((n, ci, h, w), 4242 + ci, co)
        k = po.uniform((ci, co, f, f), 4343 + ci, co)
        want = np.stack([po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8) for i in range(n)])
        print(f"{ci}->{co} {h}x{w} f{f} n{n} (K={ci * f * f})", flush=True)
        report("ffma", ffma_conv(x, k), want)
        report("tf32x1", tf32_conv(x, k), want)
        for mode in ("trunc", "rne"):
            xh, xl = split(x, mode)
            kh, kl = split(k, mode)
            t_main = tf32_conv(xh, kh)
            t_corr = tf32_conv(xh, kl) + tf32_conv(xl, kh)
            report(f"3x-{mode}", t_main + t_corr, want)


if __name__ == "__main__":
    main()
