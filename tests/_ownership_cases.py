"""Write-ownership cases, run by tests/test_gpu_ownership.py in a subprocess
with DCONV_LIB = paper_1809_10170_b200/libdconv_b200_own.so (the
DCONV_DEBUG_OWNERSHIP build): every conv kernel store of an output element
counts itself, and each case asserts that every element of the output view
-- padded channel slots included -- was written exactly once and nothing
else (halo ring, blocks outside a C_o range) was written at all.  The GPU
analogue of the reference's debug ownership map.

Covers: the three FFMA CTA tiles, forced split-K ks = 2..16 (DSMEM
reduction), the tail-split launch, the epilogue-warpgroup hand-off, skip-add
and fused max-pool epilogues, C_o block ranges with peer stores, the
first-layer reader, the generic kernel, and the TF32 / split-TF32
tensor-core kernels (stacked 7x7 tiles, strided space-to-depth reads)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1809_10170_b200 import _abi, nets  # noqa: E402

L = _abi.lib()
assert "_own" in _abi.LIB_PATH, _abi.LIB_PATH
RESULTS = []


def _region(act: nets.Act, b0=0, nb=None):
    """Expected counts: 1 on the interior of blocks [b0, b0+nb), else 0."""
    want = torch.zeros(act.buf.shape, dtype=torch.int32, device="cuda")
    nb = nets.nblk(act.c) - b0 if nb is None else nb
    h = act.halo
    want[:, b0:b0 + nb, h:h + act.h, h:h + act.w, :] = 1
    return want


def case(name, out: nets.Act, run, b0=0, nb=None):
    counts = torch.zeros(out.buf.numel(), dtype=torch.int32, device="cuda")
    _abi.check(L.dconv_debug_set_ownership(counts.data_ptr(), out.buf.data_ptr(),
                                           out.buf.numel()))
    try:
        run()
        torch.cuda.synchronize()
    finally:
        _abi.check(L.dconv_debug_set_ownership(None, None, 0))
    got = counts.view(out.buf.shape)
    want = _region(out, b0, nb)
    bad = int((got != want).sum())
    mx = int(got.max())
    RESULTS.append((name, bad, mx))
    assert bad == 0, f"{name}: {bad} elements written != expected (max count {mx})"


def act_in(n, c, h, w, seed):
    a = nets.Act(n, c, h, w)
    nets._fill(a.buf, seed, 1)
    return a


def weights(l, seed):
    wd = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), device="cuda")
    nets._fill(wd, seed, 2)
    return nets.pack_weights(wd, l.first)


def main():
    shapes = [(64, 64, 58, 58, 3, 1, 2), (24, 40, 17, 23, 5, 1, 3), (200, 24, 9, 9, 3, 2, 4),
              (96, 72, 13, 31, 1, 2, 2), (512, 136, 16, 16, 3, 1, 2)]
    for t, (ci, co, hi, wi, f, s, n) in enumerate(shapes):
        l = nets.Layer(f"c{t}", ci, co, hi, wi, f, f, s)
        x, w = act_in(n, ci, hi, wi, 10 + t), weights(l, 20 + t)
        skip = act_in(n, co, l.h_o, l.w_o, 30 + t)
        for tv in (1, 2, 3):
            for epi, sk in ((_abi.EPI_RELU, None), (_abi.EPI_ADD_RELU, skip)):
                y = nets.Act(n, co, l.h_o, l.w_o, halo=1)
                case(f"ffma tile {tv} {l} epi {epi}", y,
                     lambda: nets.conv(l, n, x, w, y, epi, sk, tile_variant=tv))
            for ks in (2, 3, 4, 8, 16):
                os.environ["DCONV_KSPLIT"] = str(ks)
                try:
                    y = nets.Act(n, co, l.h_o, l.w_o, halo=1)
                    case(f"ffma tile {tv} split-K {ks} {l}", y,
                         lambda: nets.conv(l, n, x, w, y, _abi.EPI_ADD_RELU, skip,
                                           tile_variant=tv))
                finally:
                    del os.environ["DCONV_KSPLIT"]
    # many units with a ragged last wave (tail-split launch), epilogue warpgroup
    l = nets.Layer("tail", 64, 128, 30, 30, 3, 3, 1)
    n = 37
    x, w = act_in(n, 64, 30, 30, 40), weights(l, 41)
    y = nets.Act(n, 128, 28, 28, halo=1)
    case("ffma tail split", y, lambda: nets.conv(l, n, x, w, y, _abi.EPI_RELU))
    # fused max-pool epilogue (FFMA)
    l = nets.Layer("pool", 16, 64, 34, 34, 3, 3, 1)
    x, w = act_in(2, 16, 34, 34, 50), weights(l, 51)
    for tv in (1, 2):
        z = nets.Act(2, 64, 16, 16, halo=1)
        case(f"ffma fused pool tile {tv}", z,
             lambda: nets.conv(l, 2, x, w, z, _abi.EPI_RELU | _abi.EPI_MAXPOOL, tile_variant=tv))
    # C_o block ranges (a rank's slice) with peer stores into other buffers
    l = nets.Layer("co", 64, 64, 30, 30, 3, 3, 1)
    x, w = act_in(1, 64, 30, 30, 60), weights(l, 61)
    for b0, cnt in ((0, 2), (2, 2), (6, 2), (3, 1)):
        y = nets.Act(1, 64, 28, 28, halo=1)
        peers = [nets.Act(1, 64, 28, 28, halo=1) for _ in range(3)]
        pp = [q.base() + 4 * b0 * q.blk for q in peers]
        case(f"ffma co range {b0}+{cnt} + 3 peers", y,
             lambda: nets.conv(l, 1, x, w, y.block_view(b0, cnt), _abi.EPI_RELU, None, None,
                               None, (b0, cnt), peers=pp), b0=b0, nb=cnt)
    # first-layer reader (dense image) and its C_o range / peers
    for (ci, co, hi, f, s) in ((3, 64, 226, 3, 1), (3, 64, 229, 7, 2), (3, 96, 227, 11, 4)):
        l = nets.Layer("first", ci, co, hi, hi, f, f, s, first=True)
        xd = torch.empty((2, ci, hi, hi), device="cuda")
        nets._fill(xd, 70, 1)
        w = weights(l, 71)
        y = nets.Act(2, co, l.h_o, l.w_o, halo=1)
        case(f"first layer {f}x{f}/s{s}", y, lambda: nets.conv(l, 2, xd, w, y, _abi.EPI_RELU))
    # generic kernel (c_b = 4 via the drop-in API)
    from paper_1809_10170_b200 import dconv as D
    sh = D.ConvShape(12, 20, 11, 13, 3, 3, 1)
    xb = D.pack_feature_map(torch.rand(12, 11, 13, device="cuda"), 4)
    kb = D.pack_kernel(torch.rand(12, 20, 3, 3, device="cuda"), 4, 4)
    yb = D.BlockedFeatureMap(20, sh.h_o, sh.w_o, 4, data=torch.zeros(
        (1, 5, sh.h_o, sh.w_o, 4), device="cuda"))
    counts = torch.zeros(yb.data.numel(), dtype=torch.int32, device="cuda")
    _abi.check(L.dconv_debug_set_ownership(counts.data_ptr(), yb.data.data_ptr(),
                                           yb.data.numel()))
    D.conv_direct(xb, kb, sh, D.BlockingParams(4, 1, 4), out=yb)
    torch.cuda.synchronize()
    _abi.check(L.dconv_debug_set_ownership(None, None, 0))
    assert bool((counts == 1).all()), "generic kernel"
    RESULTS.append(("generic c_b=4", 0, int(counts.max())))
    # tensor cores: TF32 and split-TF32 (stride 1, 1x1, stacked 7x7, strided)
    for x3 in (False, True):
        for (ci, co, hi, f, s, n) in ((64, 128, 30, 3, 1, 2), (256, 64, 14, 1, 1, 4),
                                      (64, 256, 9, 3, 1, 8), (64, 72, 21, 3, 2, 2),
                                      (128, 128, 15, 3, 2, 4)):
            l = nets.Layer("tc", ci, co, hi, hi, f, f, s)
            x = act_in(n, ci, hi, hi, 80)
            wp = nets.prepare_tf32(l, weights(l, 81), x3=x3)
            skip = act_in(n, co, l.h_o, l.w_o, 82)
            y = nets.Act(n, co, l.h_o, l.w_o, halo=1)
            case(f"{'tf32x3' if x3 else 'tf32'} {l}", y,
                 lambda: nets.conv_tf32(l, n, x, wp, y, _abi.EPI_ADD_RELU, skip, x3=x3))
        l = nets.Layer("tcpool", 16, 64, 34, 34, 3, 3, 1)
        x = act_in(2, 16, 34, 34, 90)
        wp = nets.prepare_tf32(l, weights(l, 91), x3=x3)
        z = nets.Act(2, 64, 16, 16, halo=1)
        case(f"{'tf32x3' if x3 else 'tf32'} fused pool", z,
             lambda: nets.conv_tf32(l, 2, x, wp, z, _abi.EPI_RELU | _abi.EPI_MAXPOOL, x3=x3))
    print(f"ownership: {len(RESULTS)} cases, every output element written exactly once")
    for name, bad, mx in RESULTS:
        print(f"  {name}: max count {mx}")


if __name__ == "__main__":
    main()
