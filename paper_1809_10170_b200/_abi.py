"""ctypes binding of the C-ABI in ``include/dconv_cuda.h``.

The shared library ``libdconv_b200.so`` (built in-tree by
``__graft_entry__.build()``) holds every CUDA kernel of the hot path.  There is
no CPU or PyTorch fallback: if the library is missing, or a call returns an
error code, the call raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DCONV_LIB") or os.path.join(_HERE, "libdconv_b200.so")  # override: A/B builds

# error codes (dconv_cuda.h)
OK, EINVAL_SHAPE, ELAYOUT, EPARAM, ECUDA, ENCCL, EUNSUPPORTED, EFORMAT, EBLOCKED, EIO = range(10)
FILE_FEATURE_MAP, FILE_KERNEL = 0, 1
EPI_NONE, EPI_RELU, EPI_ADD, EPI_ADD_RELU = range(4)
EPI_MAXPOOL = 4  # flag: fused 2x2/s2 max-pool (TF32 path)
ALGO_AUTO, ALGO_FFMA, ALGO_GENERIC, ALGO_TF32, ALGO_TF32X3 = range(5)


class ConvDesc(ctypes.Structure):
    """Mirror of ``dconv_conv_desc`` (dconv_cuda.h)."""

    _fields_ = [(n, ctypes.c_int) for n in (
        "n", "c_i", "c_o", "h_i", "w_i", "h_f", "w_f", "stride", "h_o", "w_o",
        "c_ib", "c_ob")] + [(n, ctypes.c_int64) for n in (
            "in_img_stride", "in_blk_stride", "in_row_stride",
            "out_img_stride", "out_blk_stride", "out_row_stride",
            "skip_img_stride", "skip_blk_stride", "skip_row_stride")] + [
        ("epilogue", ctypes.c_int), ("algo", ctypes.c_int),
        ("co_block_begin", ctypes.c_int), ("co_block_count", ctypes.c_int),
        ("tile_variant", ctypes.c_int)]


class FileHeader(ctypes.Structure):
    """Mirror of ``dconv_file_header`` (7 int32 words)."""

    _fields_ = [(n, ctypes.c_int32) for n in ("c", "h", "w", "c_b", "c_o", "c_ib", "kind")]


class DconvError(RuntimeError):
    """Raised for DCONV_ECUDA / DCONV_ENCCL / DCONV_EUNSUPPORTED."""


_lib: Optional[ctypes.CDLL] = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64

_SIGS = {
    "dconv_conv_desc_init": (_I, [ctypes.POINTER(ConvDesc)] + [_I] * 10),
    "dconv_conv_shape": (_I, [_I] * 7 + [ctypes.POINTER(_I)] * 2),
    "dconv_conv_flops": (_L, [_I] * 6),
    "dconv_cuda_conv_direct": (_I, [ctypes.POINTER(ConvDesc), _P, _P, _P, _P, _P]),
    "dconv_cuda_tf32_prepared_size": (_I, [ctypes.POINTER(ConvDesc), ctypes.POINTER(_L)]),
    "dconv_cuda_prepare_tf32_weights": (_I, [ctypes.POINTER(ConvDesc), _P, _P, _P]),
    "dconv_cuda_conv_direct_tf32": (_I, [ctypes.POINTER(ConvDesc), _P, _P, _P, _P, _P]),
    "dconv_cuda_tf32x3_prepared_size": (_I, [ctypes.POINTER(ConvDesc), ctypes.POINTER(_L)]),
    "dconv_cuda_prepare_tf32x3_weights": (_I, [ctypes.POINTER(ConvDesc), _P, _P, _P]),
    "dconv_cuda_conv_direct_tf32x3": (_I, [ctypes.POINTER(ConvDesc), _P, _P, _P, _P, _P]),
    "dconv_cuda_conv_first_layer": (
        _I, [ctypes.POINTER(ConvDesc), _P, _L, _P, _P, _P, _P]),
    "dconv_cuda_conv_direct_peers": (
        _I, [ctypes.POINTER(ConvDesc), _P, _P, _P, _P, ctypes.POINTER(_P), _I, _P]),
    "dconv_cuda_conv_first_layer_peers": (
        _I, [ctypes.POINTER(ConvDesc), _P, _L, _P, _P, _P, ctypes.POINTER(_P), _I, _P]),
    "dconv_cuda_pack_kernel": (_I, [_P] + [_I] * 6 + [_P, _P]),
    "dconv_cuda_unpack_kernel": (_I, [_P] + [_I] * 6 + [_P, _P]),
    "dconv_cuda_pack_feature_map": (_I, [_P] + [_I] * 6 + [_P, _P]),
    "dconv_cuda_pack_space_to_depth": (_I, [_P] + [_I] * 5 + [_P, _P]),
    "dconv_cuda_space_to_depth_blocked": (_I, [_P, _L, _L, _L] + [_I] * 5 + [_P, _P]),
    "dconv_cuda_unpack_feature_map": (_I, [_P] + [_I] * 6 + [_P, _P]),
    "dconv_cuda_relu_blocked": (_I, [_P, _L, _P]),
    "dconv_cuda_add_blocked": (_I, [_P, _P, _P, _L, _I, _P]),
    "dconv_cuda_maxpool2x2_blocked": (_I, [_P] + [_I] * 5 + [_P, _L, _L, _L, _P]),
    "dconv_cuda_zero": (_I, [_P, _L, _P]),
    "dconv_cuda_launch_count": (_L, []),
    "dconv_cuda_ffma_cluster_slots": (_I, [_I, _I, _P, _P]),
    "dconv_debug_set_ownership": (_I, [_P, _P, _L]),
    "dconv_cuda_fp32_peak_probe": (ctypes.c_double, [_P]),
    "dconv_cuda_ffma2_pattern_probe": (ctypes.c_double, [_P]),
    "dconv_file_payload_floats": (_L, [ctypes.POINTER(FileHeader)]),
    "dconv_file_read_header": (_I, [ctypes.c_char_p, ctypes.POINTER(FileHeader)]),
    "dconv_file_read_payload": (_I, [ctypes.c_char_p, _P, _L]),
    "dconv_file_write": (_I, [ctypes.c_char_p, ctypes.POINTER(FileHeader), _P, _L]),
    "dconv_pack_kernel_file": (_I, [ctypes.c_char_p, _I, _I, ctypes.c_char_p]),
    "dconv_cuda_load_kernel_file": (_I, [ctypes.c_char_p, _I, _I, _P, _P]),
    "dconv_cuda_strerror": (ctypes.c_char_p, [_I]),
    "dconv_cuda_last_error_detail": (ctypes.c_char_p, []),
}

EXPORTED = tuple(_SIGS)


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DconvError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() first "
                "(there is no CPU fallback for the hot path)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI return code to the reference's exception types.

    EINVAL_SHAPE / ELAYOUT / EPARAM / EFORMAT / EBLOCKED -> ValueError
    (std::invalid_argument in the reference: shape.cpp:26, tensor.cpp:29,
    reference.cpp:28; "parse error" / "already blocked");
    ECUDA / ENCCL / EUNSUPPORTED / EIO -> DconvError (std::runtime_error)."""
    if rc == OK:
        return
    l = lib()
    msg = f"{l.dconv_cuda_strerror(rc).decode()}: {l.dconv_cuda_last_error_detail().decode()}"
    if rc in (EINVAL_SHAPE, ELAYOUT, EPARAM, EFORMAT, EBLOCKED):
        raise ValueError(msg)
    raise DconvError(msg)


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
