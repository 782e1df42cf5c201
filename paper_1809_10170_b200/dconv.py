"""The reference ``dconv`` operator API, device-resident, over the C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(``/root/reference/proj/core/include/dconv/{shape,tensor,model}.hpp`` and the
``direct`` module of SPEC.md:283-372), so parity tests read like the
reference's own.  Tensors live in HBM as torch CUDA tensors (torch is only the
allocator/stream provider); every operation is a kernel of
``libdconv_b200.so``.  The C++ twin of this API is ``include/dconv/*.hpp``.

Differences from the reference, all additive:
  * an optional outermost batch dimension ``n`` (SPEC.md:132 is batch 1); each
    image slice is byte-identical to the reference BlockedFeatureMap;
  * ``conv_direct`` takes fused-epilogue options (ReLU / skip-add) and an
    optional preallocated output (SPEC.md:308 describes one).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch

from . import _abi
from ._abi import check, lib, ptr, stream_ptr

_layout_transforms = 0


def layout_transform_count() -> int:
    """Process-wide count of pack/unpack calls (tensor.hpp:156-159)."""
    return _layout_transforms


def _bump() -> None:
    global _layout_transforms
    _layout_transforms += 1


def round_up(value: int, block: int) -> int:  # tensor.hpp:28-30
    return (value + block - 1) // block * block


class ConvShape:
    """Valid-convolution geometry (shape.hpp:29-45, shape.cpp:30-40).

    Raises ValueError("ConvShape: ...") exactly where the reference throws
    std::invalid_argument."""

    __slots__ = ("c_i", "c_o", "h_i", "w_i", "h_f", "w_f", "stride", "h_o", "w_o")

    def __init__(self, ci: int, co: int, hi: int, wi: int, hf: int, wf: int,
                 s: int = 1):
        import ctypes
        ho, wo = ctypes.c_int(0), ctypes.c_int(0)
        check(lib().dconv_conv_shape(ci, co, hi, wi, hf, wf, s,
                                     ctypes.byref(ho), ctypes.byref(wo)))
        self.c_i, self.c_o, self.h_i, self.w_i = ci, co, hi, wi
        self.h_f, self.w_f, self.stride = hf, wf, s
        self.h_o, self.w_o = ho.value, wo.value

    def __eq__(self, other) -> bool:
        return isinstance(other, ConvShape) and all(
            getattr(self, k) == getattr(other, k) for k in self.__slots__)

    def __repr__(self) -> str:
        return (f"ConvShape({self.c_i}, {self.c_o}, {self.h_i}, {self.w_i}, "
                f"{self.h_f}, {self.w_f}, s={self.stride})")


def conv_flops(shape: ConvShape) -> int:
    """2*c_i*c_o*h_o*w_o*h_f*w_f (reference.cpp:106-109)."""
    return int(lib().dconv_conv_flops(shape.c_i, shape.c_o, shape.h_o,
                                      shape.w_o, shape.h_f, shape.w_f))


@dataclass(frozen=True)
class BlockingParams:
    """(c_ob, w_ob, c_ib) of model.hpp:54-61.  On the GPU c_ob/c_ib fix the
    blocked layout; w_ob (the CPU register-tile width) is accepted and
    recorded but the CUDA kernels choose their own pixel tiles."""
    c_ob: int = 8
    w_ob: int = 1
    c_ib: int = 8


class BlockedFeatureMap:
    """Channel-blocked map (tensor.hpp:50-81) with an optional batch dim.

    ``data`` is a CUDA tensor of shape [n, padded_channels/c_b, h, w, c_b]."""

    def __init__(self, c: int, h: int, w: int, cb: int, n: int = 1,
                 data: Optional[torch.Tensor] = None, device=None):
        if not (c >= 1 and h >= 1 and w >= 1):
            raise ValueError("BlockedFeatureMap: dims must be >= 1")
        if cb < 1:
            raise ValueError("BlockedFeatureMap: block size must be >= 1")
        if n < 1:
            raise ValueError("BlockedFeatureMap: batch must be >= 1")
        self.channels, self.height, self.width, self.c_b, self.n = c, h, w, cb, n
        self.padded_channels = round_up(c, cb)
        shape = (n, self.padded_channels // cb, h, w, cb)
        if data is None:
            data = torch.zeros(shape, dtype=torch.float32,
                               device=device or torch.device("cuda"))
        elif tuple(data.shape) != shape or data.dtype != torch.float32:
            raise ValueError(f"BlockedFeatureMap: data must be float32 {shape}")
        self.data = data

    def block_count(self) -> int:
        return self.padded_channels // self.c_b

    def block_elems(self) -> int:
        return self.height * self.width * self.c_b

    def offset(self, c: int, y: int, x: int) -> int:  # tensor.hpp:71-74
        return (c // self.c_b) * self.block_elems() + (y * self.width + x) * self.c_b + c % self.c_b


class BlockedKernel:
    """Blocked weights [c_o/c_ob][c_i/c_ib][h_f][w_f][c_ib][c_ob]
    (tensor.hpp:105-141)."""

    def __init__(self, ci: int, co: int, hf: int, wf: int, cob: int, cib: int,
                 data: Optional[torch.Tensor] = None, device=None):
        if not (ci >= 1 and co >= 1 and hf >= 1 and wf >= 1):
            raise ValueError("BlockedKernel: dims must be >= 1")
        if cob < 1 or cib < 1:
            raise ValueError("BlockedKernel: block sizes must be >= 1")
        self.c_i, self.c_o, self.h_f, self.w_f = ci, co, hf, wf
        self.c_ob, self.c_ib = cob, cib
        self.padded_c_i, self.padded_c_o = round_up(ci, cib), round_up(co, cob)
        shape = (self.padded_c_o // cob, self.padded_c_i // cib, hf, wf, cib, cob)
        if data is None:
            data = torch.zeros(shape, dtype=torch.float32,
                               device=device or torch.device("cuda"))
        self.data = data

    def in_blocks(self) -> int:
        return self.padded_c_i // self.c_ib

    def out_blocks(self) -> int:
        return self.padded_c_o // self.c_ob

    def slab_elems(self) -> int:
        return self.h_f * self.w_f * self.c_ib * self.c_ob

    def offset(self, jb, ib, n, m, ii, jj) -> int:  # tensor.hpp:131-137
        return (((((jb * self.in_blocks() + ib) * self.h_f + n) * self.w_f + m)
                 * self.c_ib + ii) * self.c_ob + jj)


def pack_feature_map(src: torch.Tensor, c_b: int, stream=None) -> BlockedFeatureMap:
    """pack_feature_map (tensor.cpp:65-73) on the device; src is [c,h,w] or
    [n,c,h,w] float32 CUDA.  Bit-exact; padded channels are exact zeros."""
    _bump()
    s4 = src if src.dim() == 4 else src.unsqueeze(0)
    s4 = s4.contiguous()
    n, c, h, w = s4.shape
    out = BlockedFeatureMap(c, h, w, c_b, n=n, device=src.device,
                            data=torch.empty((n, round_up(c, c_b) // c_b, h, w, c_b),
                                             dtype=torch.float32, device=src.device))
    check(lib().dconv_cuda_pack_feature_map(ptr(s4), n, c, h, w, c_b, 0,
                                            ptr(out.data), stream_ptr(stream)))
    return out


def unpack_feature_map(src: BlockedFeatureMap, stream=None) -> torch.Tensor:
    """unpack_feature_map (tensor.cpp:75-83): [n, c, h, w] dense, padding dropped."""
    _bump()
    out = torch.empty((src.n, src.channels, src.height, src.width),
                      dtype=torch.float32, device=src.data.device)
    check(lib().dconv_cuda_unpack_feature_map(ptr(src.data), src.n, src.channels,
                                              src.height, src.width, src.c_b, 0,
                                              ptr(out), stream_ptr(stream)))
    return out


def pack_kernel(src: torch.Tensor, c_ob: int, c_ib: int, stream=None) -> BlockedKernel:
    """pack_kernel (tensor.cpp:85-95): dense [c_i][c_o][h_f][w_f] -> blocked."""
    _bump()
    src = src.contiguous()
    ci, co, hf, wf = src.shape
    k = BlockedKernel(ci, co, hf, wf, c_ob, c_ib, device=src.device)
    check(lib().dconv_cuda_pack_kernel(ptr(src), ci, co, hf, wf, c_ob, c_ib,
                                       ptr(k.data), stream_ptr(stream)))
    return k


def unpack_kernel(src: BlockedKernel, stream=None) -> torch.Tensor:
    """unpack_kernel (tensor.cpp:97-108)."""
    _bump()
    out = torch.empty((src.c_i, src.c_o, src.h_f, src.w_f), dtype=torch.float32,
                      device=src.data.device)
    check(lib().dconv_cuda_unpack_kernel(ptr(src.data), src.c_i, src.c_o, src.h_f,
                                         src.w_f, src.c_ob, src.c_ib, ptr(out),
                                         stream_ptr(stream)))
    return out


def make_desc(shape: ConvShape, n: int, c_ib: int, c_ob: int,
              epilogue: int = _abi.EPI_NONE, algo: int = _abi.ALGO_AUTO
              ) -> _abi.ConvDesc:
    d = _abi.ConvDesc()
    import ctypes
    check(lib().dconv_conv_desc_init(ctypes.byref(d), n, shape.c_i, shape.c_o,
                                     shape.h_i, shape.w_i, shape.h_f, shape.w_f,
                                     shape.stride, c_ib, c_ob))
    d.epilogue = epilogue
    d.algo = algo
    return d


def _check_map(m: BlockedFeatureMap, shape: ConvShape, c_b: int, n: int, what: str) -> None:
    """A caller-supplied output / skip map must have the output geometry (the
    C++ overload's checks, dropin.cpp): otherwise the kernel would write or
    read past the end of its buffer."""
    if (m.channels, m.height, m.width) != (shape.c_o, shape.h_o, shape.w_o):
        raise ValueError(f"conv: {what} dims do not match shape")
    if m.c_b != c_b:
        raise ValueError(f"conv_direct: layout error ({what} c_b != c_ob)")
    if m.n != n:
        raise ValueError(f"conv: {what} batch does not match input")
    need = n * (round_up(shape.c_o, c_b) // c_b) * shape.h_o * shape.w_o * c_b
    if m.data.numel() < need or not m.data.is_contiguous():
        raise ValueError(f"conv: {what} buffer too small or not contiguous")


def conv_direct(inp: BlockedFeatureMap, kernel: BlockedKernel, shape: ConvShape,
                params: BlockingParams, workers: int = 0, *,
                relu: bool = False, skip: Optional[BlockedFeatureMap] = None,
                out: Optional[BlockedFeatureMap] = None,
                algo: int = _abi.ALGO_AUTO, tile_variant: int = 0,
                stream=None) -> BlockedFeatureMap:
    """conv_direct: blocked in (c_b == c_ib) x blocked
    kernel (c_ob, c_ib) -> blocked out (c_b == c_ob).  ``workers`` is the
    reference's CPU thread count; on the GPU the grid replaces the pool and
    the result is bitwise independent of it.  ``tile_variant``
    picks the FFMA CTA tile (dconv_conv_desc.tile_variant; 0 = selector)."""
    if inp.c_b != params.c_ib or kernel.c_ib != params.c_ib:
        raise ValueError("conv_direct: layout error (input c_b / kernel c_ib "
                         "must equal params.c_ib)")
    if kernel.c_ob != params.c_ob:
        raise ValueError("conv_direct: layout error (kernel c_ob != params.c_ob)")
    if (inp.channels, inp.height, inp.width) != (shape.c_i, shape.h_i, shape.w_i):
        raise ValueError("conv: input dims do not match shape")
    if (kernel.c_i, kernel.c_o, kernel.h_f, kernel.w_f) != (
            shape.c_i, shape.c_o, shape.h_f, shape.w_f):
        raise ValueError("conv: kernel dims do not match shape")
    if skip is not None:
        _check_map(skip, shape, params.c_ob, inp.n, "skip")
    if out is not None:
        _check_map(out, shape, params.c_ob, inp.n, "output")
    epi = (_abi.EPI_RELU if relu else 0) | (_abi.EPI_ADD if skip is not None else 0)
    d = make_desc(shape, inp.n, params.c_ib, params.c_ob, epi, algo)
    d.tile_variant = tile_variant
    if out is None:
        out = BlockedFeatureMap(shape.c_o, shape.h_o, shape.w_o, params.c_ob,
                                n=inp.n, device=inp.data.device,
                                data=torch.empty((inp.n, round_up(shape.c_o, params.c_ob) // params.c_ob,
                                                  shape.h_o, shape.w_o, params.c_ob),
                                                 dtype=torch.float32, device=inp.data.device))
    import ctypes
    check(lib().dconv_cuda_conv_direct(ctypes.byref(d), ptr(inp.data), ptr(kernel.data),
                                       ptr(skip.data if skip is not None else None),
                                       ptr(out.data), stream_ptr(stream)))
    return out


class PreparedKernel:
    """A blocked kernel rearranged once into the tensor-core operand layout
    (the C++ ``dconv::cuda::DevicePreparedKernel``): ``split=True`` holds the
    hi/lo halves of the split-TF32 kernel (the fp32 tolerance of
    ``conv_direct``), ``split=False`` the single-pass TF32 layout."""

    def __init__(self, kernel: BlockedKernel, shape: ConvShape, split: bool = True,
                 stream=None):
        import ctypes
        if kernel.c_ob != 8 or kernel.c_ib != 8:
            raise ValueError("conv_direct: layout error (tensor-core path needs c_b = 8)")
        if (kernel.c_i, kernel.c_o, kernel.h_f, kernel.w_f) != (
                shape.c_i, shape.c_o, shape.h_f, shape.w_f):
            raise ValueError("conv: kernel dims do not match shape")
        self.shape, self.split = shape, split
        d = make_desc(shape, 1, 8, 8)
        sz = ctypes.c_int64(0)
        L = lib()
        size_fn = L.dconv_cuda_tf32x3_prepared_size if split else L.dconv_cuda_tf32_prepared_size
        prep_fn = L.dconv_cuda_prepare_tf32x3_weights if split else L.dconv_cuda_prepare_tf32_weights
        check(size_fn(ctypes.byref(d), ctypes.byref(sz)))
        self.data = torch.empty(sz.value, dtype=torch.float32, device=kernel.data.device)
        check(prep_fn(ctypes.byref(d), ptr(kernel.data), ptr(self.data), stream_ptr(stream)))


def conv_direct_tc(inp: BlockedFeatureMap, kernel: PreparedKernel, *, relu: bool = False,
                   skip: Optional[BlockedFeatureMap] = None,
                   out: Optional[BlockedFeatureMap] = None, stream=None) -> BlockedFeatureMap:
    """conv_direct on the tcgen05 tensor cores (c_b = 8; any k x k stride-s
    layer with s <= 8 -- stride-s layers are computed over the space-to-depth
    view of the input, read in place): the split-TF32 kernel for a
    ``PreparedKernel(split=True)`` (fp32 tolerance), else one TF32 pass
    (looser tolerance)."""
    import ctypes
    shape = kernel.shape
    if inp.c_b != 8:
        raise ValueError("conv_direct: layout error (tensor-core path needs c_b = 8)")
    if (inp.channels, inp.height, inp.width) != (shape.c_i, shape.h_i, shape.w_i):
        raise ValueError("conv: input dims do not match shape")
    if skip is not None:
        _check_map(skip, shape, 8, inp.n, "skip")
    if out is not None:
        _check_map(out, shape, 8, inp.n, "output")
    epi = (_abi.EPI_RELU if relu else 0) | (_abi.EPI_ADD if skip is not None else 0)
    d = make_desc(shape, inp.n, 8, 8, epi,
                  _abi.ALGO_TF32X3 if kernel.split else _abi.ALGO_TF32)
    if out is None:
        out = BlockedFeatureMap(shape.c_o, shape.h_o, shape.w_o, 8, n=inp.n,
                                device=inp.data.device,
                                data=torch.empty((inp.n, round_up(shape.c_o, 8) // 8,
                                                  shape.h_o, shape.w_o, 8),
                                                 dtype=torch.float32, device=inp.data.device))
    L = lib()
    fn = L.dconv_cuda_conv_direct_tf32x3 if kernel.split else L.dconv_cuda_conv_direct_tf32
    check(fn(ctypes.byref(d), ptr(inp.data), ptr(kernel.data),
             ptr(skip.data if skip is not None else None), ptr(out.data), stream_ptr(stream)))
    return out


def relu_blocked(x: BlockedFeatureMap, stream=None) -> BlockedFeatureMap:
    """relu_blocked, in place; padding stays 0."""
    check(lib().dconv_cuda_relu_blocked(ptr(x.data), x.data.numel(), stream_ptr(stream)))
    return x


def add_blocked(a: BlockedFeatureMap, b: BlockedFeatureMap, relu: bool = False,
                out: Optional[BlockedFeatureMap] = None, stream=None) -> BlockedFeatureMap:
    """Skip layer: element-wise a + b (optionally ReLU)."""
    if a.data.shape != b.data.shape:
        raise ValueError("add_blocked: layout error (maps differ)")
    if out is None:
        out = BlockedFeatureMap(a.channels, a.height, a.width, a.c_b, n=a.n,
                                device=a.data.device, data=torch.empty_like(a.data))
    check(lib().dconv_cuda_add_blocked(ptr(a.data), ptr(b.data), ptr(out.data),
                                       a.data.numel(), int(relu), stream_ptr(stream)))
    return out


def maxpool2x2_blocked(x: BlockedFeatureMap, stream=None) -> BlockedFeatureMap:
    """2x2 stride-2 max-pool within each channel pencil."""
    out = BlockedFeatureMap(x.channels, x.height // 2, x.width // 2, x.c_b, n=x.n,
                            device=x.data.device,
                            data=torch.empty((x.n, x.block_count(), x.height // 2,
                                              x.width // 2, x.c_b),
                                             dtype=torch.float32, device=x.data.device))
    check(lib().dconv_cuda_maxpool2x2_blocked(ptr(x.data), x.n, x.block_count(),
                                              x.height, x.width, x.c_b, ptr(out.data),
                                              0, 0, 0, stream_ptr(stream)))
    return out


Layer = Tuple[BlockedKernel, ConvShape, BlockingParams]


def layer_chain(inp: BlockedFeatureMap, layers: Sequence, stream=None) -> BlockedFeatureMap:
    """layer_chain: each layer's output feeds the next with
    zero layout transforms; a layer is (kernel, shape, params[, relu]).
    Raises ValueError (layout error) when c_ib(L+1) != c_ob(L)."""
    before = layout_transform_count()
    x = inp
    for idx, layer in enumerate(layers):
        kernel, shape, params = layer[:3]
        relu = bool(layer[3]) if len(layer) > 3 else False
        if x.c_b != params.c_ib:
            raise ValueError(f"layer_chain: layout error at layer {idx} "
                             f"(c_ib={params.c_ib} but previous c_ob={x.c_b})")
        x = conv_direct(x, kernel, shape, params, relu=relu, stream=stream)
    assert layout_transform_count() == before, "layout transform inside chain"
    return x


# ---------------------------------------------------------------- tensor files
# SPEC.md:129 (7-int header + little-endian fp32 payload) and the CLI `pack`
# step SPEC.md:580-587; the header word order is documented in dconv_cuda.h.
def _host_f32(t) -> "np.ndarray":
    import numpy as np
    if isinstance(t, torch.Tensor):
        t = t.detach().cpu().numpy()
    return np.ascontiguousarray(t, dtype=np.float32)


def read_header(path: str) -> _abi.FileHeader:
    h = _abi.FileHeader()
    check(lib().dconv_file_read_header(path.encode(), h))
    return h


def _write(path: str, hdr: Tuple[int, ...], payload) -> None:
    a = _host_f32(payload)
    h = _abi.FileHeader(*hdr)
    check(lib().dconv_file_write(path.encode(), h, a.ctypes.data, a.size))


def save_feature_map(path: str, dense) -> None:
    """Dense [c][h][w] map -> file (c_b = 0)."""
    c, hh, w = dense.shape
    _write(path, (c, hh, w, 0, 0, 0, _abi.FILE_FEATURE_MAP), dense)


def save_blocked_feature_map(path: str, x: BlockedFeatureMap) -> None:
    if x.n != 1:
        raise ValueError("tensor files hold one image (SPEC.md:132)")
    _write(path, (x.channels, x.height, x.width, x.c_b, 0, 0, _abi.FILE_FEATURE_MAP), x.data)


def save_kernel(path: str, dense) -> None:
    """Dense KernelTensor [c_i][c_o][h_f][w_f] -> file (c_ob = c_ib = 0)."""
    ci, co, hf, wf = dense.shape
    _write(path, (ci, hf, wf, 0, co, 0, _abi.FILE_KERNEL), dense)


def save_blocked_kernel(path: str, k: BlockedKernel) -> None:
    _write(path, (k.c_i, k.h_f, k.w_f, k.c_ob, k.c_o, k.c_ib, _abi.FILE_KERNEL), k.data)


def read_payload(path: str) -> Tuple[_abi.FileHeader, "np.ndarray"]:
    """Header and raw fp32 payload of a tensor file (host memory)."""
    import numpy as np
    h = read_header(path)
    out = np.empty(lib().dconv_file_payload_floats(h), dtype=np.float32)
    check(lib().dconv_file_read_payload(path.encode(), out.ctypes.data, out.size))
    return h, out


def load_kernel_file(path: str, c_ob: int, c_ib: int, stream=None) -> BlockedKernel:
    """Weight ingest: a dense or already-blocked kernel file -> device
    BlockedKernel (dense files are repacked on the GPU)."""
    h = read_header(path)
    if h.kind != _abi.FILE_KERNEL:
        raise ValueError(f"parse error: '{path}' is not a kernel file")
    k = BlockedKernel(h.c, h.c_o, h.h, h.w, c_ob, c_ib)
    check(lib().dconv_cuda_load_kernel_file(path.encode(), c_ob, c_ib, ptr(k.data),
                                            stream_ptr(stream)))
    return k


def pack_kernel_file(in_path: str, c_ob: int, c_ib: int, out_path: str) -> None:
    """The CLI `pack` subcommand: dense kernel file ->
    blocked kernel file; a blocked input raises ValueError("already blocked")."""
    check(lib().dconv_pack_kernel_file(in_path.encode(), c_ob, c_ib, out_path.encode()))
