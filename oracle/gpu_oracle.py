"""fp64 conv_oracle64 on the GPU (oracle/oracle_gpu.cu) -- TEST
INFRASTRUCTURE ONLY: the whole-output checker at the bench sizes.  Bit-exact
with the reference's conv_oracle64 (reference.cpp:70-87) after rounding to
fp32 (tests/test_oracle_gpu.py pins it against the golden fixtures)."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle_gpu.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise RuntimeError(f"{SO} not built (oracle/Makefile)")
        l = ctypes.CDLL(SO)
        P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
        l.orcg_conv_oracle64.restype = I
        l.orcg_conv_oracle64.argtypes = [P, I, I, I, I, I, L, L, L, P, I, I, I, I, P, P]
        _lib = l
    return _lib


def conv64(in_ptr: int, n: int, c_i: int, h_i: int, w_i: int, in_cb: int,
           in_img: int, in_blk: int, in_row: int, k_dense, s: int, stream=None):
    """fp64 [n][ceil(C_o/8)][H_o][W_o][8] of conv(input view, dense kernel
    [C_i][C_o][H_f][W_f] on the device).  The input is a blocked view with
    strides in floats (cb = 1: dense CHW)."""
    import torch
    c_i2, c_o, h_f, w_f = k_dense.shape
    assert c_i2 == c_i and k_dense.is_cuda and k_dense.dtype == torch.float32
    k = k_dense.contiguous()
    h_o, w_o = (h_i - h_f) // s + 1, (w_i - w_f) // s + 1
    out = torch.empty((n, (c_o + 7) // 8, h_o, w_o, 8), dtype=torch.float64, device=k.device)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    rc = lib().orcg_conv_oracle64(in_ptr, n, c_i, h_i, w_i, in_cb, in_img, in_blk, in_row,
                                  k.data_ptr(), c_o, h_f, w_f, s, out.data_ptr(), st)
    if rc:
        raise RuntimeError(f"orcg_conv_oracle64 failed ({rc})")
    return out


def conv64_act(act, l, k_dense, stream=None):
    """conv64 over a nets.Act (its whole halo'd buffer is the layer input,
    as the plans read it) or a dense [n][C][H][W] tensor (first layers)."""
    import torch
    if isinstance(act, torch.Tensor):
        n, c, h, w = act.shape
        return conv64(act.data_ptr(), n, c, h, w, 1, c * h * w, h * w, w, k_dense, l.s, stream)
    ptr, img, blk, row = act.full_view()
    return conv64(ptr, act.n, l.c_i, l.h_i, l.w_i, 8, img, blk, row, k_dense, l.s, stream)


def check_tol(got, want64, atol=1e-4, rtol=1e-5):
    """Per element |got - want| <= atol + rtol*|want| with want rounded to
    fp32 (what conv_oracle64 returns).  Returns (ok, n_bad, max_err, worst
    ratio err / bound)."""
    import torch
    want = want64.float().double()
    err = (got.double() - want).abs()
    bound = atol + rtol * want.abs()
    ratio = float((err / bound).max()) if err.numel() else 0.0
    nbad = int((err > bound).sum())
    return nbad == 0, nbad, float(err.max()) if err.numel() else 0.0, ratio
