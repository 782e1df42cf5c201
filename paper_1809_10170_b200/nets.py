"""Layer catalogs of the BASELINE.json configs and the zero-reshape chain
executor (``layer_chain``, widened with halo'd buffers,
fused ReLU / skip-add epilogues and max-pool).

Every activation lives in the blocked layout with c_b = 8 from the first
layer's output to the network output: the only layout transform in a network
is the first-layer *reader* (which consumes the dense image directly, no pack).
"Pre-padded" inputs (BASELINE.json) are halo'd buffers: a producer writes its
output into the interior of the consumer's buffer through the C-ABI's view
strides, and the halo ring is zeroed once at allocation, outside any timing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import torch

from . import _abi
from ._abi import check, lib, ptr, stream_ptr

CB = 8  # channel block of every activation and weight in the networks


@dataclass(frozen=True)
class Layer:
    """One conv layer: ConvShape fields (shape.hpp:29-45) + its role."""
    name: str
    c_i: int
    c_o: int
    h_i: int
    w_i: int
    h_f: int
    w_f: int
    s: int = 1
    first: bool = False  # reads the dense network input (first-layer reader)

    @property
    def h_o(self) -> int:
        return (self.h_i - self.h_f) // self.s + 1

    @property
    def w_o(self) -> int:
        return (self.w_i - self.w_f) // self.s + 1

    @property
    def flops(self) -> int:  # conv_flops, reference.cpp:106-109 (one image)
        return 2 * self.c_i * self.c_o * self.h_o * self.w_o * self.h_f * self.w_f

    def in_bytes(self) -> int:
        return 4 * self.c_i * self.h_i * self.w_i

    def out_bytes(self) -> int:
        return 4 * self.c_o * self.h_o * self.w_o

    def w_bytes(self) -> int:
        return 4 * self.c_i * self.c_o * self.h_f * self.w_f


CFG1 = [Layer("cfg1", 64, 64, 58, 58, 3, 3, 1)]

ALEXNET = [
    Layer("conv1", 3, 96, 227, 227, 11, 11, 4, first=True),
    Layer("conv2", 96, 256, 31, 31, 5, 5, 1),
    Layer("conv3", 256, 384, 15, 15, 3, 3, 1),
    Layer("conv4", 384, 384, 15, 15, 3, 3, 1),
    Layer("conv5", 384, 256, 15, 15, 3, 3, 1),
]

VGG16 = [
    Layer("conv1_1", 3, 64, 226, 226, 3, 3, 1, first=True),
    Layer("conv1_2", 64, 64, 226, 226, 3, 3, 1),
    Layer("conv2_1", 64, 128, 114, 114, 3, 3, 1),
    Layer("conv2_2", 128, 128, 114, 114, 3, 3, 1),
    Layer("conv3_1", 128, 256, 58, 58, 3, 3, 1),
    Layer("conv3_2", 256, 256, 58, 58, 3, 3, 1),
    Layer("conv3_3", 256, 256, 58, 58, 3, 3, 1),
    Layer("conv4_1", 256, 512, 30, 30, 3, 3, 1),
    Layer("conv4_2", 512, 512, 30, 30, 3, 3, 1),
    Layer("conv4_3", 512, 512, 30, 30, 3, 3, 1),
    Layer("conv5_1", 512, 512, 16, 16, 3, 3, 1),
    Layer("conv5_2", 512, 512, 16, 16, 3, 3, 1),
    Layer("conv5_3", 512, 512, 16, 16, 3, 3, 1),
]
# a 2x2/s2 max-pool follows these VGG layers (224->112->56->28->14)
VGG16_POOL_AFTER = {"conv1_2", "conv2_2", "conv3_3", "conv4_3"}

GOOGLENET = [
    Layer("conv1_7x7_s2", 3, 64, 229, 229, 7, 7, 2, first=True),
    Layer("inc3a_1x1", 192, 64, 28, 28, 1, 1, 1),
    Layer("inc3a_3x3", 96, 128, 30, 30, 3, 3, 1),
    Layer("inc3a_5x5", 16, 32, 32, 32, 5, 5, 1),
    Layer("inc4a_1x1", 480, 192, 14, 14, 1, 1, 1),
    Layer("inc4a_3x3", 112, 224, 16, 16, 3, 3, 1),
]


def resnet50_layers() -> List[Tuple[str, Layer]]:
    """ResNet-50 v1.5-style topology (stride on the 3x3; projection shortcut
    on the first block of each stage).  Stem input 229 instead of BASELINE's
    230: (230 - 7) % 2 != 0 is rejected by ConvShape (shape.cpp:36)."""
    out = [("stem", Layer("stem", 3, 64, 229, 229, 7, 7, 2, first=True))]
    spatial, c_in = 56, 64
    for stage, (mid, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        c_out = mid * 4
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            h_in = spatial
            h_mid = h_in // stride
            tag = f"s{stage + 1}b{b + 1}"
            out.append((tag, Layer(f"{tag}_c1", c_in, mid, h_in, h_in, 1, 1, 1)))
            if stride == 1:
                out.append((tag, Layer(f"{tag}_c2", mid, mid, h_in + 2, h_in + 2, 3, 3, 1)))
            else:
                out.append((tag, Layer(f"{tag}_c2", mid, mid, h_in + 1, h_in + 1, 3, 3, 2)))
            out.append((tag, Layer(f"{tag}_c3", mid, c_out, h_mid, h_mid, 1, 1, 1)))
            if b == 0:
                crop = h_in - 1 if stride == 2 else h_in
                out.append((tag, Layer(f"{tag}_proj", c_in, c_out, crop, crop, 1, 1, stride)))
            c_in = c_out
            spatial = h_mid
    return out


CONFIGS: Dict[str, List[Layer]] = {
    "cfg1": CFG1,
    "alexnet": ALEXNET,
    "vgg16": VGG16,
    "googlenet": GOOGLENET,
    "resnet50": [l for _, l in resnet50_layers()],
}


def network_flops(layers: List[Layer]) -> int:
    return sum(l.flops for l in layers)


# ---------------------------------------------------------------- execution
def _desc(l: Layer, n: int, epilogue: int = 0) -> _abi.ConvDesc:
    d = _abi.ConvDesc()
    check(lib().dconv_conv_desc_init(ctypes.byref(d), n, l.c_i, l.c_o, l.h_i, l.w_i,
                                     l.h_f, l.w_f, l.s, CB, CB))
    d.epilogue = epilogue
    return d


def nblk(c: int) -> int:
    return (c + CB - 1) // CB


class Act:
    """A blocked activation buffer [n][nblk][H+2h][W+2h][8] with a view of its
    interior (offset and strides in floats)."""

    def __init__(self, n: int, c: int, h: int, w: int, halo: int = 0,
                 pad_hi_only: bool = False, device="cuda"):
        self.n, self.c, self.h, self.w, self.halo = n, c, h, w, halo
        self.pad_hi_only = pad_hi_only
        # pad_hi_only: halo on top/left only (ResNet stride-2 "pad 1/0")
        hp = h + (halo if pad_hi_only else 2 * halo)
        wp = w + (halo if pad_hi_only else 2 * halo)
        self.hp, self.wp = hp, wp
        self.buf = torch.zeros((n, nblk(c), hp, wp, CB), dtype=torch.float32, device=device)
        self.row = wp * CB
        self.blk = hp * self.row
        self.img = nblk(c) * self.blk
        self.off = (halo * wp + halo) * CB

    def base(self) -> int:
        """Interior element (0, 0, 0): where a producer writes."""
        return self.buf.data_ptr() + 4 * self.off

    def full_view(self):
        """(ptr, img, blk, row) of the whole halo'd buffer: what a consumer
        conv reads (its h_i/w_i include the halo)."""
        return (self.buf.data_ptr(), self.img, self.blk, self.row)

    def interior(self) -> torch.Tensor:
        return self.buf[:, :, self.halo:self.halo + self.h, self.halo:self.halo + self.w, :]

    def block_view(self, b0: int, count: Optional[int] = None) -> "Act":
        """The same map seen from output block b0 on (a rank's C_o slice of
        ``count`` blocks inside the full buffer): base() moves, strides stay,
        and the view's channel count covers only its blocks."""
        import copy
        v = copy.copy(self)
        v.off = self.off + b0 * self.blk
        nb = nblk(self.c) - b0 if count is None else count
        v.c = max(0, min(self.c - b0 * CB, nb * CB))
        return v

    def clone_zeros(self) -> "Act":
        """Same geometry, fresh zeroed buffer (halo ring and padding 0)."""
        return Act(self.n, self.c, self.h, self.w, halo=self.halo, pad_hi_only=self.pad_hi_only,
                   device=self.buf.device)


def conv(l: Layer, n: int, x: "Act|torch.Tensor", w: torch.Tensor, out: Act,
         epilogue: int = 0, skip: Optional[Act] = None, stream=None,
         in_view: Optional[Tuple[int, int, int, int]] = None,
         co_range: Optional[Tuple[int, int]] = None, tile_variant: int = 0,
         peers: Optional[List[int]] = None) -> None:
    """Launch one conv layer through the C-ABI.  ``x`` is an Act (blocked) or,
    for a first layer, the dense [n][c][h][w] network input.  ``in_view``
    optionally overrides (ptr, img, blk, row) of the blocked input (crops).
    ``co_range`` = (first block, block count) computes only those output
    blocks into ``out`` (a rank's C_o slice); ``skip`` is then read from the
    same blocks of the full skip map.  ``peers``: device addresses (P2P-mapped
    peer copies of ``out``) that receive the same stores -- the fused
    C_o-shard gather."""
    d = _desc(l, n, epilogue)
    d.tile_variant = tile_variant
    d.out_img_stride, d.out_blk_stride, d.out_row_stride = out.img, out.blk, out.row
    b0 = 0
    if co_range is not None:
        b0, d.co_block_count = co_range
        d.co_block_begin = b0
    sp = 0
    if skip is not None:
        d.skip_img_stride, d.skip_blk_stride, d.skip_row_stride = skip.img, skip.blk, skip.row
        sp = skip.base() + 4 * b0 * skip.blk
    st = stream_ptr(stream)
    pl = (ctypes.c_void_p * max(1, len(peers or [])))(*(peers or []))
    np_ = len(peers or [])
    if l.first:
        if np_:
            check(lib().dconv_cuda_conv_first_layer_peers(ctypes.byref(d), ptr(x), 0, ptr(w), sp,
                                                          out.base(), pl, np_, st))
        else:
            check(lib().dconv_cuda_conv_first_layer(ctypes.byref(d), ptr(x), 0, ptr(w), sp,
                                                    out.base(), st))
        return
    if in_view is None:
        in_view = x.full_view()
    d.in_img_stride, d.in_blk_stride, d.in_row_stride = in_view[1:]
    if np_:
        check(lib().dconv_cuda_conv_direct_peers(ctypes.byref(d), in_view[0], ptr(w), sp,
                                                 out.base(), pl, np_, st))
    else:
        check(lib().dconv_cuda_conv_direct(ctypes.byref(d), in_view[0], ptr(w), sp,
                                           out.base(), st))


def conv_tf32(l: Layer, n: int, x: "Act", wprep: torch.Tensor, out: Act,
              epilogue: int = 0, skip: Optional[Act] = None, stream=None,
              in_view: Optional[Tuple[int, int, int, int]] = None, x3: bool = False) -> None:
    """tcgen05/TMEM TF32 launch of a blocked layer (any k x k stride-s layer,
    s <= 8: strided layers run over the space-to-depth view of the input,
    read in place; weights prepared by prepare_tf32).  ``x3``: the split-TF32 kernel
    (fp32 tolerance; weights prepared with ``x3=True``)."""
    d = _desc(l, n, epilogue)
    d.out_img_stride, d.out_blk_stride, d.out_row_stride = out.img, out.blk, out.row
    if in_view is None:
        in_view = x.full_view()
    d.in_img_stride, d.in_blk_stride, d.in_row_stride = in_view[1:]
    sp = 0
    if skip is not None:
        d.skip_img_stride, d.skip_blk_stride, d.skip_row_stride = skip.img, skip.blk, skip.row
        sp = skip.base()
    fn = lib().dconv_cuda_conv_direct_tf32x3 if x3 else lib().dconv_cuda_conv_direct_tf32
    check(fn(ctypes.byref(d), in_view[0], ptr(wprep), sp, out.base(), stream_ptr(stream)))


def prepare_tf32(l: Layer, w_blocked: torch.Tensor, stream=None, x3: bool = False) -> torch.Tensor:
    """One-time rearrangement of a blocked kernel into the UMMA operand layout
    (``x3``: hi/lo operand pairs for the split-TF32 kernel)."""
    d = _desc(l, 1)
    sz = ctypes.c_int64(0)
    L = lib()
    size_fn = L.dconv_cuda_tf32x3_prepared_size if x3 else L.dconv_cuda_tf32_prepared_size
    prep_fn = L.dconv_cuda_prepare_tf32x3_weights if x3 else L.dconv_cuda_prepare_tf32_weights
    check(size_fn(ctypes.byref(d), ctypes.byref(sz)))
    out = torch.empty(sz.value, dtype=torch.float32, device=w_blocked.device)
    check(prep_fn(ctypes.byref(d), ptr(w_blocked), ptr(out), stream_ptr(stream)))
    return out


def maxpool_into(x: Act, out: Act, stream=None, out_ptr: Optional[int] = None) -> None:
    """2x2/s2 max-pool of x into the view ``out`` (``out_ptr`` overrides its
    base address: a peer's copy of the same view)."""
    check(lib().dconv_cuda_maxpool2x2_blocked(x.base(), x.n, nblk(x.c), x.h, x.w, CB,
                                              out.base() if out_ptr is None else out_ptr,
                                              out.img, out.blk, out.row, stream_ptr(stream)))


def pack_weights(dense: torch.Tensor, first: bool, stream=None) -> torch.Tensor:
    """Dense [c_i][c_o][h_f][w_f] -> blocked (c_ob = 8; c_ib = 8, or c_i for
    a first layer).  The one-time repack kernel (tensor.cpp:85-95)."""
    ci, co, hf, wf = dense.shape
    cib = ci if first else CB
    out = torch.empty((nblk(co), (ci + cib - 1) // cib, hf, wf, cib, CB),
                      dtype=torch.float32, device=dense.device)
    check(lib().dconv_cuda_pack_kernel(ptr(dense.contiguous()), ci, co, hf, wf, CB, cib,
                                       ptr(out), stream_ptr(stream)))
    return out


@dataclass
class Step:
    """One launch of a plan: a conv layer (kind 'conv' / 'first'), a
    layout-preserving op ('pool') or a collective ('gather')."""
    fn: object
    name: str
    kind: str
    flops: int = 0      # algorithmic FLOPs of this launch on this rank
    layer: Optional[Layer] = None
    bytes: int = 0      # compulsory HBM bytes of this launch (the roofline's other axis)


def conv_bytes(l: Layer, n: int, epilogue: int = 0) -> int:
    """Compulsory bytes of one conv launch over n images: input
    read once, output written once (a quarter with the fused 2x2 pool), the
    skip map read once with an ADD epilogue, the weights read once (unpadded
    channel counts)."""
    out = l.c_o * l.h_o * l.w_o
    if epilogue & _abi.EPI_MAXPOOL:
        out //= 4
    skip = l.c_o * l.h_o * l.w_o if epilogue & _abi.EPI_ADD else 0
    return 4 * (n * (l.c_i * l.h_i * l.w_i + out + skip) + l.c_i * l.c_o * l.h_f * l.w_f)


def pool_bytes(a: "Act") -> int:
    """2x2/s2 max-pool of a map: read it once, write a quarter."""
    return 4 * a.n * a.c * a.h * a.w * 5 // 4


def _on_stream(st):
    """Context that makes torch's current stream the plan's launch stream
    (collectives and symmetric-memory barriers are enqueued on the current
    stream; the conv kernels on the stream a step is given)."""
    import contextlib
    if st is None:
        return contextlib.nullcontext()
    if isinstance(st, torch.cuda.Stream):
        return torch.cuda.stream(st)
    return torch.cuda.stream(torch.cuda.ExternalStream(int(st)))


def _sm_count() -> int:
    """SMs of the current device (148 on B200; the CPU tests have no GPU)."""
    if torch.cuda.is_available():
        return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return 148


# tensor-core plans: "tf32" (one TF32 pass, looser tolerance) and "tf32x3"
# (split-TF32, the fp32 tolerance of the FFMA path)
TC_ALGOS = ("tf32", "tf32x3")


@dataclass
class Plan:
    """A network instantiated on one device: weights, activations, and the
    ordered launch list.  ``run()`` is one step (one pass over the batch).

    ``shard`` = (rank, world, group) selects batch-1 output-block sharding:
    every conv computes this rank's contiguous j' range into a local slice,
    ReLU / skip-add / max-pool run on the slice, and an all-gather of the
    slices rebuilds the full (halo'd) blocked map for the next layer."""
    name: str
    n: int
    layers: List[Layer]
    shard: Optional[Tuple[int, int, object]] = None
    algo: str = "ffma"   # "tf32" / "tf32x3": blocked layers on the tcgen05 path
    # C_o-shard exchange: "nccl" = slice + all-gather; "peer" = the conv/pool
    # epilogue stores into every rank's full map (symmetric memory over
    # NVLink) followed by a device barrier -- no collective on the data path.
    # Emulation of all `world` ranks on one device (tests, bench parity; the
    # ranks' launches run one after another, nothing waits on another rank):
    # "emulate" = every rank's launches of a layer (its C_o slice, the same
    # kernel configuration a real rank runs) into one full map -- what the
    # all-gather assembles; "emulate_peer" = every rank keeps its own full
    # map and its conv / pool epilogues also store into the other ranks'
    # copies (peer stores into local buffers, the fused-gather addressing).
    gather_mode: str = "nccl"
    weights: Dict[str, torch.Tensor] = field(default_factory=dict)
    tiles: Dict[str, int] = field(default_factory=dict)  # autotuned FFMA CTA tile per layer
    steps: List = field(default_factory=list)
    input: Optional[torch.Tensor] = None   # dense network input (first layer)
    output: Optional[Act] = None

    @property
    def x3(self) -> bool:
        return self.algo == "tf32x3"
    per_layer_inputs: Dict[str, Act] = field(default_factory=dict)
    outputs: Dict[str, Act] = field(default_factory=dict)

    @property
    def flops(self) -> int:
        """Algorithmic FLOPs this rank executes per step."""
        return sum(s.flops for s in self.steps)

    def run(self, stream=None) -> None:
        for st in self.steps:
            st.fn(stream)

    def autotune(self, stream=None, variants=(1, 2, 3), reps: int = 3) -> Dict[str, int]:
        """Times every FFMA conv step with each CTA tile (desc.tile_variant)
        and keeps the fastest -- the GPU analogue of the reference's autotune
        (model.hpp:103-109), run once at plan build, outside
        any timed region.  The layers are timed IN the step: whole passes of
        the plan with every layer on the same tile, events around each conv
        launch, the fastest of the repeats.  (A layer repeated on its own
        finds its 50 MB input in L2 and preferred, for the VGG 28x28 layers, a
        tile that is 5% slower behind its producer in the chain.)"""
        s = stream or torch.cuda.current_stream()
        allowed = {}
        for st in self.steps:
            if st.kind != "conv":
                continue
            # the 256 px x 32 ch tile only where 64-channel groups leave one
            # half empty (C_o = 32, 224, ...)
            l = st.layer
            allowed[st.name] = tuple(variants) + (
                (4,) if l is not None and l.c_o % 64 and 4 not in variants else ())
        best: Dict[str, Tuple[float, int]] = {}
        for v in sorted({v for vs in allowed.values() for v in vs}):
            for name, vs in allowed.items():
                if v in vs:
                    self.tiles[name] = v
            for r in range(reps + 1):
                evs = []
                for st in self.steps:
                    if st.kind == "conv" and v in allowed[st.name]:
                        a = torch.cuda.Event(enable_timing=True)
                        b = torch.cuda.Event(enable_timing=True)
                        a.record(s)
                        st.fn(s)
                        b.record(s)
                        evs.append((st.name, a, b))
                    else:
                        st.fn(s)
                s.synchronize()
                if r == 0:
                    continue  # warm-up pass
                for name, a, b in evs:
                    ms = a.elapsed_time(b)
                    if name not in best or ms < best[name][0]:
                        best[name] = (ms, v)
        for name, (_, v) in best.items():
            self.tiles[name] = v
        return dict(self.tiles)

    def io_inputs(self) -> List[torch.Tensor]:
        """Device tensors that are the step's inputs (network input, or every
        layer's own input for the independent-layer configs)."""
        ins = [self.input] if self.input is not None else []
        return ins + [a.buf for a in self.per_layer_inputs.values()]

    def io_outputs(self) -> List[torch.Tensor]:
        if self.per_layer_inputs:
            return [a.buf for a in self.outputs.values()]
        return [self.output.buf]

    def io_map(self):
        """(inputs, outputs): [(device tensor, index of the step that reads it
        last)] and [(device tensor, index of the step that writes it)] -- the
        points after which a streamed batch may refill an input buffer, and
        before which the previous batch's result must have left."""
        names = [s.name for s in self.steps]
        ins = []
        if self.input is not None:  # read by the first launch (a reader or a repack)
            ins.append((self.input, 0))
        for name, a in self.per_layer_inputs.items():
            ins.append((a.buf, names.index(name)))
        if self.per_layer_inputs:
            outs = [(a.buf, names.index(name)) for name, a in self.outputs.items()]
        else:
            outs = [(self.output.buf, len(self.steps) - 1)]
        return ins, outs

    # -- building blocks ----------------------------------------------------
    def _local(self, full: Act, c: int) -> Act:
        return Act(self.n, c, full.h, full.w, halo=full.halo, pad_hi_only=full.pad_hi_only,
                   device=full.buf.device)

    def _adopt_symmetric(self, full: Act) -> None:
        """Move ``full`` into symmetric memory (one allocation per rank,
        P2P-mapped) and record the peers' addresses of the same map."""
        if getattr(full, "symm", None) is not None:
            return
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        rank, world, group = self.shard
        group = group or dist.group.WORLD
        t = symm_mem.empty(tuple(full.buf.shape), dtype=torch.float32, device=full.buf.device)
        t.zero_()  # halo ring and padded channels are zeros on every rank
        h = symm_mem.rendezvous(t, group)
        off = t.data_ptr() - h.buffer_ptrs[rank]
        full.buf = t
        full.symm = h
        full.peer_bases = [h.buffer_ptrs[r] + off for r in range(world) if r != rank]

    def _peer_ptrs(self, full: Act, b0: int) -> List[int]:
        """Peers' addresses of block b0's interior origin in ``full``."""
        return [b + 4 * (full.off + b0 * full.blk) for b in full.peer_bases]

    def _barrier(self, name: str, full: Act) -> None:
        h = full.symm

        def run(st):
            with _on_stream(st):  # ordered after this rank's stores on the plan's stream
                h.barrier(channel=0)
        self.steps.append(Step(run, f"barrier_{name}", "barrier"))

    def _gather(self, name: str, full: Act, local: Act) -> None:
        from .shard import all_gather_blocks
        group = self.shard[2]

        def run(st):
            with _on_stream(st):  # NCCL enqueues on the current stream: the plan's
                all_gather_blocks(full.buf[0], local.buf[0], group)
        self.steps.append(Step(run, f"gather_{name}", "gather"))

    def conv_into(self, l: Layer, x, y: Act, epilogue: int = 0, skip: Optional[Act] = None,
                  gather: bool = True, in_view=None) -> Act:
        """conv(l) into y (or into this rank's slice of y, then gathered).
        Returns the Act holding this rank's result (y, or the slice)."""
        w = self.weights[l.name]
        kind = "first" if l.first else "conv"
        if self.shard is None:
            tc = self.algo in TC_ALGOS and not (self.x3 and self._few_units(l, epilogue))
            if tc and l.first and l.s > 1 and in_view is None:
                return self._tf32_s2d_first(l, x, y, epilogue, skip)
            # (stride-1 first layers -- VGG conv1_1 -- run on the FFMA
            # first-layer reader below in the tensor-core plans too: it reads
            # the dense image in place, where the tcgen05 kernel would need a
            # channel-padded copy of it, and is as fast: 0.14 ms against
            # 0.03 ms pack + 0.14 ms split-TF32 at VGG b32)
            if tc and not l.first:
                # stride 1, 1x1 of any stride, and k x k stride s (the C-ABI
                # reads the space-to-depth view of the input in place)
                wp = prepare_tf32(l, w, x3=self.x3)
                self.weights[l.name + ".tf32"] = wp
                self.steps.append(Step(lambda st: conv_tf32(l, self.n, x, wp, y, epilogue, skip, st,
                                                            in_view, x3=self.x3),
                                       l.name, "tf32", self.n * l.flops, l,
                                       conv_bytes(l, self.n, epilogue)))
                return y
            self.steps.append(Step(lambda st: conv(l, self.n, x, w, y, epilogue, skip, st, in_view,
                                                   tile_variant=self.tiles.get(l.name, 0)),
                                   l.name, kind, self.n * l.flops, l,
                                   conv_bytes(l, self.n, epilogue)))
            return y
        from .shard import block_range
        rank, world, _ = self.shard
        if self.n != 1:
            raise ValueError("C_o sharding is the batch-1 mode")
        if self.gather_mode in ("emulate", "emulate_peer"):
            return self._conv_emulated(l, x, y, epilogue, skip, in_view, kind)
        b0, cnt = block_range(nblk(l.c_o), world, rank)
        flops = l.flops * min(cnt * CB, l.c_o - b0 * CB) // l.c_o
        if self.gather_mode == "peer" and gather:
            # fused gather: this rank's blocks go straight into every rank's
            # full map (local store + NVLink peer stores), then one barrier
            self._adopt_symmetric(y)
            yv, peers = y.block_view(b0, cnt), self._peer_ptrs(y, b0)
            self.steps.append(Step(lambda st: conv(l, self.n, x, w, yv, epilogue, skip, st,
                                                   in_view, (b0, cnt),
                                                   tile_variant=self.tiles.get(l.name, 0),
                                                   peers=peers),
                                   l.name, kind, flops, l))
            self._barrier(l.name, y)
            return yv
        ys = self._local(y, cnt * CB)
        self.steps.append(Step(lambda st: conv(l, self.n, x, w, ys, epilogue, skip, st, in_view,
                                               (b0, cnt), tile_variant=self.tiles.get(l.name, 0)),
                               l.name, kind, flops, l))
        if gather:
            self._gather(l.name, y, ys)
        return ys

    @staticmethod
    def _copies(a: Act, world: int) -> List[Act]:
        """emulate_peer: rank r's own full copy of map ``a`` (copy 0 is ``a``)."""
        if getattr(a, "copies", None) is None:
            a.copies = [a] + [a.clone_zeros() for _ in range(world - 1)]
        return a.copies

    def _conv_emulated(self, l: Layer, x, y: Act, epilogue: int, skip: Optional[Act],
                       in_view, kind: str) -> Act:
        """Every rank's launch of layer ``l`` on this device, rank by rank."""
        from .shard import block_range
        _, world, _ = self.shard
        w = self.weights[l.name]
        peer_mode = self.gather_mode == "emulate_peer"
        ys = self._copies(y, world) if peer_mode else [y] * world
        xs = (self._copies(x, world) if peer_mode and isinstance(x, Act) else [x] * world)
        sks = (self._copies(skip, world) if peer_mode and skip is not None else [skip] * world)
        for r in range(world):
            b0, cnt = block_range(nblk(l.c_o), world, r)
            flops = l.flops * min(cnt * CB, l.c_o - b0 * CB) // l.c_o
            yv = ys[r].block_view(b0, cnt)
            peers = [ys[q].base() + 4 * b0 * ys[q].blk for q in range(world) if q != r] \
                if peer_mode else None
            iv = in_view
            if in_view is not None and xs[r] is not x:
                iv = (xs[r].buf.data_ptr() + (in_view[0] - x.buf.data_ptr()),) + tuple(in_view[1:])
            self.steps.append(Step(
                lambda st, xr=xs[r], yv=yv, skr=sks[r], iv=iv, b0=b0, cnt=cnt, peers=peers:
                conv(l, self.n, xr, w, yv, epilogue, skr, st, iv, (b0, cnt),
                     tile_variant=self.tiles.get(l.name, 0), peers=peers),
                f"{l.name}@r{r}", kind, flops, l))
        return y

    def _few_units(self, l: Layer, epilogue: int) -> bool:
        """Split-TF32 plans run a layer on the FFMA kernel (same fp32
        tolerance) when it has fewer tensor-core work units (128-pixel
        M-tiles x 128-channel groups) than SMs: batch-1 layers, where the FFMA
        kernel's split-K over a cluster keeps every SM busy and the split-TF32
        kernel (no split-K) would leave most of them idle."""
        if epilogue & _abi.EPI_MAXPOOL:
            return False
        units = self.n * -(-l.h_o // 16) * -(-l.w_o // 8) * -(-l.c_o // 128)
        return units < _sm_count()

    def _tf32_s2d_first(self, l: Layer, x, y: Act, epilogue: int, skip) -> Act:
        """TF32 path, stride-f first layer (GoogLeNet/ResNet 7x7/s2, AlexNet
        11x11/s4): space-to-depth turns it into a stride-1 conv with f*f*C_i
        channels and a ceil(h_f/f) x ceil(w_f/f) filter (exact: the extra taps
        and channels are zero weights), run on the tcgen05 kernel.  FLOPs are
        counted with the original layer."""
        f = l.s
        cs = l.c_i * f * f
        hs, ws = -(-l.h_i // f), -(-l.w_i // f)
        hf, wf = -(-l.h_f // f), -(-l.w_f // f)
        lb = Layer(l.name, cs, l.c_o, hs, ws, hf, wf, 1, False)
        assert (lb.h_o, lb.w_o) == (l.h_o, l.w_o)
        w = self.weights[l.name]
        dense = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), dtype=torch.float32, device=w.device)
        check(lib().dconv_cuda_unpack_kernel(ptr(w), l.c_i, l.c_o, l.h_f, l.w_f, CB, l.c_i,
                                             ptr(dense), stream_ptr(None)))
        # w_s2d[(dy*f + dx)*C_i + c][o][n'][m'] = w[c][o][f*n' + dy][f*m' + dx]
        wpad = torch.zeros((l.c_i, l.c_o, hf * f, wf * f), dtype=torch.float32, device=w.device)
        wpad[:, :, :l.h_f, :l.w_f] = dense
        ws2d = (wpad.view(l.c_i, l.c_o, hf, f, wf, f).permute(3, 5, 0, 1, 2, 4)
                .reshape(cs, l.c_o, hf, wf).contiguous())
        wp = prepare_tf32(lb, pack_weights(ws2d, False), x3=self.x3)
        self.weights[l.name + ".tf32"] = wp
        xb = Act(self.n, cs, hs, ws, device=w.device)
        n = self.n
        self.steps.append(Step(
            lambda st: check(lib().dconv_cuda_pack_space_to_depth(
                ptr(x), n, l.c_i, l.h_i, l.w_i, f, ptr(xb.buf), stream_ptr(st))),
            f"pack_{l.name}", "pack", bytes=4 * n * (l.c_i * l.h_i * l.w_i + cs * hs * ws)))
        self.steps.append(Step(lambda st: conv_tf32(lb, n, xb, wp, y, epilogue, skip, st,
                                                    x3=self.x3),
                               l.name, "tf32", n * l.flops, l, conv_bytes(lb, n, epilogue)))
        return y

    def pool_into(self, name: str, src_local: Act, z: Act) -> None:
        """2x2/s2 max-pool of this rank's result into z (gathered if sharded)."""
        if self.shard is None or self.gather_mode == "emulate":
            # (emulate: src_local is the full map every rank's conv wrote;
            # pooling it equals pooling the slices -- max is exact)
            self.steps.append(Step(lambda st: maxpool_into(src_local, z, st), name, "pool",
                                   bytes=pool_bytes(src_local)))
            return
        if self.gather_mode == "emulate_peer":
            from .shard import block_range
            _, world, _ = self.shard
            srcs, zs = self._copies(src_local, world), self._copies(z, world)
            for r in range(world):
                b0, cnt = block_range(nblk(z.c), world, r)
                src, zv = srcs[r].block_view(b0, cnt), zs[r].block_view(b0, cnt)
                peers = [zs[q].base() + 4 * b0 * zs[q].blk for q in range(world) if q != r]

                def pool_all(st, src=src, zv=zv, peers=peers):
                    maxpool_into(src, zv, st)
                    for pp in peers:
                        maxpool_into(src, zv, st, out_ptr=pp)
                self.steps.append(Step(pool_all, f"{name}@r{r}", "pool"))
            return
        if self.gather_mode == "peer":
            # pool this rank's slice into every rank's z (local + peers)
            from .shard import block_range
            rank, world, _ = self.shard
            b0, cnt = block_range(nblk(z.c), world, rank)
            self._adopt_symmetric(z)
            zv, peers = z.block_view(b0, cnt), self._peer_ptrs(z, b0)

            def pool_all(st, src=src_local, zv=zv, peers=peers):
                maxpool_into(src, zv, st)
                for pp in peers:
                    maxpool_into(src, zv, st, out_ptr=pp)
            self.steps.append(Step(pool_all, name, "pool"))
            self._barrier(name, z)
            return
        zs = self._local(z, src_local.c)
        self.steps.append(Step(lambda st: maxpool_into(src_local, zs, st), name, "pool"))
        self._gather(name, z, zs)


class Pipeline:
    """Streams batches through a plan the way a server would: the host->device
    copy of batch i+1 (pinned host buffers, a copy stream) starts as soon as
    batch i's kernels have consumed that input buffer, and the device->host
    copy of batch i's result overlaps batch i+1's kernels; only the first
    copy in and the last copy out are exposed.  Every batch still moves all
    of its bytes both ways.  Synchronisation is by CUDA events on three
    streams (compute, copy in, copy out); the plan's own buffers are reused
    (an input buffer is refilled only after its consuming launch, an output
    buffer overwritten only after its previous copy-out)."""

    def __init__(self, plan: Plan, host_inputs: List[torch.Tensor],
                 host_outputs: List[torch.Tensor], stream=None):
        self.plan = plan
        self.ins, self.outs = plan.io_map()
        if len(host_inputs) != len(self.ins) or len(host_outputs) != len(self.outs):
            raise ValueError("Pipeline: one host buffer per plan input / output")
        self.h_in, self.h_out = host_inputs, host_outputs
        self.compute = stream or torch.cuda.Stream()
        self.copy_in, self.copy_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        self.in_ready = [ev() for _ in self.ins]      # H2D of the current batch done
        self.in_free = [ev() for _ in self.ins]       # its consumer launch done
        self.out_ready = [ev() for _ in self.outs]    # producer launch done
        self.out_free = [ev() for _ in self.outs]     # D2H of the previous batch done
        self.consumer = {i: k for k, (_, i) in enumerate(self.ins)}
        self.producer = {i: k for k, (_, i) in enumerate(self.outs)}

    def _h2d(self, k: int, after_consumer: bool) -> None:
        with torch.cuda.stream(self.copy_in):
            if after_consumer:
                self.copy_in.wait_event(self.in_free[k])
            self.ins[k][0].copy_(self.h_in[k], non_blocking=True)
            self.in_ready[k].record(self.copy_in)

    def run(self, batches: int) -> None:
        """Enqueue `batches` batches (asynchronous; synchronise the streams or
        `done()` to wait)."""
        for k in range(len(self.ins)):
            self._h2d(k, after_consumer=False)
        for b in range(batches):
            for i, st in enumerate(self.plan.steps):
                if i in self.consumer:
                    self.compute.wait_event(self.in_ready[self.consumer[i]])
                if i in self.producer and b > 0:
                    self.compute.wait_event(self.out_free[self.producer[i]])
                st.fn(self.compute)
                if i in self.consumer:
                    k = self.consumer[i]
                    self.in_free[k].record(self.compute)
                    if b + 1 < batches:
                        self._h2d(k, after_consumer=True)
                if i in self.producer:
                    k = self.producer[i]
                    self.out_ready[k].record(self.compute)
                    with torch.cuda.stream(self.copy_out):
                        self.copy_out.wait_event(self.out_ready[k])
                        self.h_out[k].copy_(self.outs[k][0], non_blocking=True)
                        self.out_free[k].record(self.copy_out)

    def streams(self):
        return self.compute, self.copy_in, self.copy_out


def _fill(t: torch.Tensor, seed: int, stream_id: int, scale: float = 1.0) -> None:
    """Seeded uniform[-1,1) on the device, same counter-based generator as
    the CPU checker (oracle/oracle.c) so CPU and GPU inputs agree."""
    from .synth import fill_uniform_
    fill_uniform_(t, seed, stream_id, scale)


def build_plan(config: str, n: int, seed: int = 1809, device="cuda",
               dense_weights: Optional[Dict[str, torch.Tensor]] = None,
               shard: Optional[Tuple[int, int, object]] = None, algo: str = "ffma",
               gather_mode: str = "nccl") -> Plan:
    """Instantiates a BASELINE.json config on the current device.  ``shard``
    = (rank, world, process group) for batch-1 C_o-block sharding, with the
    exchange ``gather_mode`` "nccl" (all-gather) or "peer" (fused peer stores
    + barrier); ``algo`` = "tf32" runs the stride-1 blocked layers on the
    tcgen05 TF32 kernel."""
    if gather_mode not in ("nccl", "peer", "emulate", "emulate_peer"):
        raise ValueError(f"gather_mode {gather_mode!r}")
    layers = CONFIGS[config]
    p = Plan(config, n, list(layers), shard=shard, algo=algo, gather_mode=gather_mode)
    for idx, l in enumerate(layers):
        wd = dense_weights[l.name] if dense_weights else None
        if wd is None:
            wd = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), dtype=torch.float32, device=device)
            scale = 1.0
            if config == "resnet50":  # keep 53 unnormalised layers finite: sqrt(3/K)
                scale = (3.0 / (l.c_i * l.h_f * l.w_f)) ** 0.5
            _fill(wd, seed, 1000 + 2 * idx, scale)
        p.weights[l.name] = pack_weights(wd, l.first)
    if config in ("vgg16",):
        _build_vgg(p, device, seed)
    elif config == "resnet50":
        _build_resnet(p, device, seed)
    else:
        _build_independent(p, device, seed)
    return p


def _build_independent(p: Plan, device, seed: int) -> None:
    """AlexNet / GoogLeNet / cfg1: every layer on its own seeded input (the
    configs give pre-padded per-layer input sizes)."""
    for idx, l in enumerate(p.layers):
        if l.first:
            x = torch.empty((p.n, l.c_i, l.h_i, l.w_i), dtype=torch.float32, device=device)
            _fill(x, seed, 2 * idx)
            p.input = x
        else:
            x = Act(p.n, l.c_i, l.h_i, l.w_i, device=device)
            _fill(x.buf, seed, 2 * idx)
            _zero_pad_channels(x, l.c_i)
            p.per_layer_inputs[l.name] = x
        y = Act(p.n, l.c_o, l.h_o, l.w_o, device=device)
        p.outputs[l.name] = y
        p.conv_into(l, x, y)
    p.output = p.outputs[p.layers[-1].name]


def _zero_pad_channels(a: Act, c: int) -> None:
    if c % CB:
        a.buf[:, -1, :, :, c % CB:] = 0.0


def _build_vgg(p: Plan, device, seed: int) -> None:
    """VGG-16: conv+ReLU chain; each conv writes into the interior of the next
    conv's halo buffer (pad 1), pooling writes into the next halo buffer."""
    layers = p.layers
    x0 = torch.empty((p.n, 3, 226, 226), dtype=torch.float32, device=device)
    _fill(x0, seed, 0)
    # VGG's zero padding of the image: the 224x224 image sits in a 226 ring
    x0[:, :, 0, :] = 0; x0[:, :, -1, :] = 0; x0[:, :, :, 0] = 0; x0[:, :, :, -1] = 0
    p.input = x0
    cur = x0
    for i, l in enumerate(layers):
        last = i == len(layers) - 1
        pool = l.name in VGG16_POOL_AFTER
        # FFMA: the fused pool epilogue (conv_ffma EPI_MAXPOOL) ties the
        # separate pencil pool kernel on VGG b32 (54.28 vs 54.29 TFLOP/s) and
        # loses with the untuned tile choice, so it is opt-in
        fuse_ffma = (p.algo == "ffma" and l.w_o % 16 == 0 and l.h_o % 2 == 0
                     and os.environ.get("DCONV_POOL_FUSION") is not None)
        if pool and (p.algo in TC_ALGOS or fuse_ffma) and p.shard is None and not l.first:
            # conv + ReLU + 2x2 max-pool in one kernel, straight into the next
            # layer's halo buffer (the full-resolution map is never written).
            # FFMA: only where the pool-compatible tiles (TW a multiple of
            # the pixel-group count) cover the row without waste.
            z = Act(p.n, l.c_o, l.h_o // 2, l.w_o // 2, halo=1, device=device)
            p.outputs[l.name] = z
            p.conv_into(l, cur, z, epilogue=_abi.EPI_RELU | _abi.EPI_MAXPOOL)
            cur = z
            continue
        y = Act(p.n, l.c_o, l.h_o, l.w_o, halo=0 if (last or pool) else 1, device=device)
        p.outputs[l.name] = y
        mine = p.conv_into(l, cur, y, epilogue=_abi.EPI_RELU, gather=not pool)
        if pool:
            z = Act(p.n, l.c_o, l.h_o // 2, l.w_o // 2, halo=1, device=device)
            p.pool_into(f"pool_{l.name}", mine, z)
            cur = z
        else:
            cur = y
    p.output = cur


def _build_resnet(p: Plan, device, seed: int) -> None:
    """ResNet-50 chain: stem conv+ReLU -> 2x2 max-pool -> 16 bottlenecks with
    the skip-add + ReLU fused into the third conv's epilogue."""
    named = resnet50_layers()
    stem = named[0][1]
    x0 = torch.empty((p.n, 3, 229, 229), dtype=torch.float32, device=device)
    _fill(x0, seed, 0)
    p.input = x0
    x = Act(p.n, 64, 56, 56, device=device)
    if p.algo in TC_ALGOS and p.shard is None:
        # tcgen05 stem (space-to-depth) with ReLU + 2x2 max-pool in its epilogue
        p.outputs["stem"] = x
        p.conv_into(stem, x0, x, epilogue=_abi.EPI_RELU | _abi.EPI_MAXPOOL)
    else:
        s_out = Act(p.n, 64, 112, 112, device=device)
        p.outputs["stem"] = s_out
        mine = p.conv_into(stem, x0, s_out, epilogue=_abi.EPI_RELU, gather=False)
        p.pool_into("pool_stem", mine, x)
    blocks: Dict[str, List[Layer]] = {}
    for tag, l in named[1:]:
        blocks.setdefault(tag, []).append(l)
    for tag, ls in blocks.items():
        c1, c2, c3 = ls[0], ls[1], ls[2]
        proj = ls[3] if len(ls) > 3 else None
        mid1 = Act(p.n, c1.c_o, c1.h_o, c1.w_o, halo=1, pad_hi_only=(c2.s != 1), device=device)
        mid2 = Act(p.n, c2.c_o, c2.h_o, c2.w_o, device=device)
        y = Act(p.n, c3.c_o, c3.h_o, c3.w_o, device=device)
        p.conv_into(c1, x, mid1, epilogue=_abi.EPI_RELU)
        p.conv_into(c2, mid1, mid2, epilogue=_abi.EPI_RELU)
        if proj is not None:
            sc = Act(p.n, proj.c_o, proj.h_o, proj.w_o, device=device)
            # 1x1 s2 projection reads the 55x55 (or full) crop of x: a view
            p.conv_into(proj, x, sc, in_view=x.full_view())
            skip = sc
        else:
            skip = x
        p.conv_into(c3, mid2, y, epilogue=_abi.EPI_ADD_RELU, skip=skip)
        p.outputs[tag] = y
        x = y
    p.output = x
