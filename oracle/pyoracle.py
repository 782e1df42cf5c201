"""numpy/ctypes binding of oracle/liboracle.so (C restatement of the reference
path) and oracle/_ref/libdconv_ref.so (the reference's own sources).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdconv_ref.so")

_F = ctypes.POINTER(ctypes.c_float)
_I = ctypes.c_int
_L = ctypes.c_int64

_orc = None
_ref = None


def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_F)


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        l = ctypes.CDLL(ORACLE_SO)
        l.orc_conv_shape.argtypes = [_I] * 7 + [ctypes.POINTER(_I)] * 2
        l.orc_conv_flops.restype = _L
        l.orc_conv_flops.argtypes = [_I] * 6
        l.orc_round_up.argtypes = [_I, _I]
        for f in ("orc_pack_feature_map", "orc_unpack_feature_map"):
            getattr(l, f).argtypes = [_F, _I, _I, _I, _I, _F]
        for f in ("orc_pack_kernel", "orc_unpack_kernel"):
            getattr(l, f).argtypes = [_F, _I, _I, _I, _I, _I, _I, _F]
        for f in ("orc_conv_oracle64", "orc_conv_naive"):
            getattr(l, f).argtypes = [_F, _F] + [_I] * 7 + [_F]
        l.orc_conv_oracle64_blocked.argtypes = [_F, _F] + [_I] * 11 + [_F]
        l.orc_conv_direct.argtypes = [_F, _F] + [_I] * 12 + [_F]
        l.orc_conv_direct_literal_alg3.argtypes = [_F, _F] + [_I] * 10 + [_F]
        l.orc_relu.argtypes = [_F, _L]
        l.orc_add.argtypes = [_F, _F, _F, _L]
        l.orc_maxpool2x2.argtypes = [_F, _I, _I, _I, _I, _F]
        l.orc_fill_uniform.argtypes = [_F, _L, ctypes.c_uint64, ctypes.c_uint64]
        _orc = l
    return _orc


def ref():
    """The reference's own code (None if it was never built here)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            return None
        l = ctypes.CDLL(REF_SO)
        l.ref_conv_shape.argtypes = [_I] * 7 + [ctypes.POINTER(_I)] * 2
        l.ref_conv_flops.restype = _L
        l.ref_conv_flops.argtypes = [_I] * 7
        l.ref_conv.argtypes = [_I, _F, _F] + [_I] * 7 + [_F]
        l.ref_pack_feature_map.argtypes = [_F, _I, _I, _I, _I, _F]
        l.ref_unpack_feature_map.argtypes = [_F, _I, _I, _I, _I, _F]
        l.ref_pack_kernel.argtypes = [_F, _I, _I, _I, _I, _I, _I, _F]
        l.ref_unpack_kernel.argtypes = [_F, _I, _I, _I, _I, _I, _I, _F]
        l.ref_layout_transform_count.restype = ctypes.c_uint64
        l.ref_blocked_kernel_offset.restype = ctypes.c_size_t
        l.ref_blocked_kernel_offset.argtypes = [_I] * 12
        l.ref_conv_reordered_batch.argtypes = [_F, _F] + [_I] * 9 + [_F]
        l.ref_pool_conv_direct.argtypes = [_F, _F] + [_I] * 12 + [_F]
        _ref = l
    return _ref


def round_up(v: int, b: int) -> int:
    return (v + b - 1) // b * b


def conv_shape(ci, co, hi, wi, hf, wf, s=1):
    """(h_o, w_o) or raises ValueError like ConvShape (shape.cpp:30-40)."""
    ho, wo = _I(0), _I(0)
    if orc().orc_conv_shape(ci, co, hi, wi, hf, wf, s, ctypes.byref(ho), ctypes.byref(wo)):
        raise ValueError("ConvShape: invalid geometry")
    return ho.value, wo.value


def uniform(shape, seed: int, stream: int) -> np.ndarray:
    a = np.empty(shape, dtype=np.float32)
    orc().orc_fill_uniform(_fp(a), a.size, seed, stream)
    return a


def pack_feature_map(x: np.ndarray, c_b: int) -> np.ndarray:
    c, h, w = x.shape
    out = np.empty((round_up(c, c_b) // c_b, h, w, c_b), np.float32)
    orc().orc_pack_feature_map(_fp(np.ascontiguousarray(x)), c, h, w, c_b, _fp(out))
    return out


def unpack_feature_map(b: np.ndarray, c: int) -> np.ndarray:
    nb, h, w, c_b = b.shape
    out = np.empty((c, h, w), np.float32)
    orc().orc_unpack_feature_map(_fp(np.ascontiguousarray(b)), c, h, w, c_b, _fp(out))
    return out


def pack_kernel(k: np.ndarray, c_ob: int, c_ib: int) -> np.ndarray:
    ci, co, hf, wf = k.shape
    out = np.empty((round_up(co, c_ob) // c_ob, round_up(ci, c_ib) // c_ib, hf, wf,
                    c_ib, c_ob), np.float32)
    orc().orc_pack_kernel(_fp(np.ascontiguousarray(k)), ci, co, hf, wf, c_ob, c_ib, _fp(out))
    return out


def unpack_kernel(b: np.ndarray, ci: int, co: int) -> np.ndarray:
    _, _, hf, wf, c_ib, c_ob = b.shape
    out = np.empty((ci, co, hf, wf), np.float32)
    orc().orc_unpack_kernel(_fp(np.ascontiguousarray(b)), ci, co, hf, wf, c_ob, c_ib, _fp(out))
    return out


def conv_oracle64(x: np.ndarray, k: np.ndarray, s: int) -> np.ndarray:
    ci, hi, wi = x.shape
    _, co, hf, wf = k.shape
    ho, wo = conv_shape(ci, co, hi, wi, hf, wf, s)
    out = np.empty((co, ho, wo), np.float32)
    orc().orc_conv_oracle64(_fp(np.ascontiguousarray(x)), _fp(np.ascontiguousarray(k)),
                            ci, co, hi, wi, hf, wf, s, _fp(out))
    return out


def conv_naive(x: np.ndarray, k: np.ndarray, s: int) -> np.ndarray:
    ci, hi, wi = x.shape
    _, co, hf, wf = k.shape
    ho, wo = conv_shape(ci, co, hi, wi, hf, wf, s)
    out = np.empty((co, ho, wo), np.float32)
    orc().orc_conv_naive(_fp(np.ascontiguousarray(x)), _fp(np.ascontiguousarray(k)),
                         ci, co, hi, wi, hf, wf, s, _fp(out))
    return out


def conv_oracle64_blocked(xb: np.ndarray, kb: np.ndarray, ci: int, co: int, s: int,
                          y0: int = 0, y1: int = 1 << 30) -> np.ndarray:
    """fp64 oracle on one blocked image; rows [y0, y1) of the output computed
    (others left 0).  Returns the blocked output [jb][ho][wo][c_ob]."""
    nb, hi, wi, c_ib = xb.shape
    jb_n, _, hf, wf, _, c_ob = kb.shape
    ho, wo = conv_shape(ci, co, hi, wi, hf, wf, s)
    out = np.zeros((jb_n, ho, wo, c_ob), np.float32)
    orc().orc_conv_oracle64_blocked(_fp(np.ascontiguousarray(xb)), _fp(np.ascontiguousarray(kb)),
                                    ci, co, hi, wi, hf, wf, s, c_ib, c_ob, y0, y1, _fp(out))
    return out


def conv_direct(xb: np.ndarray, kb: np.ndarray, ci: int, co: int, s: int,
                w_ob: int = 0, threads: int = 0) -> np.ndarray:
    """Restated Alg. 3 (CPU, OpenMP over (image, j')) on blocked buffers.
    xb is [n][nb][hi][wi][c_ib] (or without n)."""
    x4 = xb if xb.ndim == 5 else xb[None]
    n, nb, hi, wi, c_ib = x4.shape
    jb_n, _, hf, wf, _, c_ob = kb.shape
    ho, wo = conv_shape(ci, co, hi, wi, hf, wf, s)
    if w_ob <= 0:
        w_ob = {8: 14, 16: 7, 32: 3}.get(c_ob, 4)
    out = np.empty((n, jb_n, ho, wo, c_ob), np.float32)
    rc = orc().orc_conv_direct(_fp(np.ascontiguousarray(x4)), _fp(np.ascontiguousarray(kb)),
                               n, ci, co, hi, wi, hf, wf, s, c_ib, c_ob, w_ob, threads, _fp(out))
    if rc:
        raise ValueError("conv_direct: parameter/layout error")
    return out if xb.ndim == 5 else out[0]


def conv_direct_pool(xb: np.ndarray, kb: np.ndarray, ci: int, co: int, s: int,
                     workers: int, w_ob: int = 0, out: np.ndarray = None) -> np.ndarray:
    """The same restated Alg. 3, scheduled on the reference's own ThreadPool
    (oracle/_ref, thread_pool.cpp) with ``workers`` pool threads plus the
    caller (DCONV_THREADS = workers).  Bitwise equal to conv_direct."""
    r = ref()
    if r is None:
        raise RuntimeError("oracle/_ref/libdconv_ref.so was not built")
    x4 = xb if xb.ndim == 5 else xb[None]
    n, nb, hi, wi, c_ib = x4.shape
    jb_n, _, hf, wf, _, c_ob = kb.shape
    ho, wo = conv_shape(ci, co, hi, wi, hf, wf, s)
    if w_ob <= 0:
        w_ob = {8: 14, 16: 7, 32: 3}.get(c_ob, 4)
    if out is None:
        out = np.empty((n, jb_n, ho, wo, c_ob), np.float32)
    rc = r.ref_pool_conv_direct(_fp(np.ascontiguousarray(x4)), _fp(np.ascontiguousarray(kb)),
                                n, ci, co, hi, wi, hf, wf, s, c_ib, c_ob, w_ob, workers, _fp(out))
    if rc:
        raise ValueError("conv_direct: parameter/layout error")
    return out if xb.ndim == 5 else out[0]


def within_tol(got: np.ndarray, want: np.ndarray, atol=1e-4, rtol=1e-5):
    """BASELINE.json tolerance |a-b| <= atol + rtol*|b| per element.
    Returns (ok, n_bad, max_abs_err)."""
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    bad = err > atol + rtol * np.abs(want.astype(np.float64))
    return (not bad.any()), int(bad.sum()), float(err.max() if err.size else 0.0)
