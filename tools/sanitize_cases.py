"""Small launches of every kernel path for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per gpurun call): FFMA CTA tiles with the
epilogue-warpgroup hand-off, forced split-K ks = 2..16 (DSMEM push
reduction, cluster mbarriers), the tail-split launch, fused pool, C_o range
+ peer stores, the first-layer reader, the TF32 / split-TF32 tcgen05 kernels
(TMEM chunk hand-off, stacked tiles, strided space-to-depth TMA), and the
layout kernels.  Prints a checksum per case."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1809_10170_b200 import _abi, nets  # noqa: E402


def act(n, c, h, w, seed, halo=0):
    a = nets.Act(n, c, h, w, halo=halo)
    nets._fill(a.buf, seed, 1)
    return a


def wts(l, seed):
    wd = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), device="cuda")
    nets._fill(wd, seed, 2)
    return nets.pack_weights(wd, l.first)


def done(name, y):
    torch.cuda.synchronize()
    print(f"{name}: sum {float(y.buf.double().sum()):.6e}", flush=True)


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    l = nets.Layer("a", 64, 64, 18, 18, 3, 3, 1)
    x, w = act(2, 64, 18, 18, 1), wts(l, 2)
    sk = act(2, 64, 16, 16, 3)
    if only in ("", "ffma"):
        for tv in (1, 2, 3):
            y = nets.Act(2, 64, 16, 16, halo=1)
            nets.conv(l, 2, x, w, y, _abi.EPI_ADD_RELU, sk, tile_variant=tv)
            done(f"ffma tile {tv}", y)
        for ks in (2, 3, 4, 8, 16):
            os.environ["DCONV_KSPLIT"] = str(ks)
            y = nets.Act(2, 64, 16, 16, halo=1)
            nets.conv(l, 2, x, w, y, _abi.EPI_ADD_RELU, sk, tile_variant=2)
            del os.environ["DCONV_KSPLIT"]
            done(f"ffma split-K {ks}", y)
        lt = nets.Layer("t", 64, 64, 10, 10, 3, 3, 1)
        xt, wt = act(150, 64, 10, 10, 4), wts(lt, 5)
        y = nets.Act(150, 64, 8, 8)
        nets.conv(lt, 150, xt, wt, y, _abi.EPI_RELU)
        done("ffma many units + tail split", y)
        z = nets.Act(2, 64, 8, 8, halo=1)
        nets.conv(l, 2, x, w, z, _abi.EPI_RELU | _abi.EPI_MAXPOOL, tile_variant=2)
        done("ffma fused pool", z)
        y = nets.Act(1, 64, 16, 16, halo=1)
        peers = [nets.Act(1, 64, 16, 16, halo=1) for _ in range(2)]
        nets.conv(l, 1, x, w, y.block_view(2, 2), _abi.EPI_RELU, None, None, None, (2, 2),
                  peers=[q.base() + 8 * q.blk for q in peers])
        done("ffma co range + peers", y)
    if only in ("", "first"):
        lf = nets.Layer("f", 3, 64, 37, 37, 7, 7, 2, first=True)
        xd = torch.empty((2, 3, 37, 37), device="cuda")
        nets._fill(xd, 6, 1)
        y = nets.Act(2, 64, lf.h_o, lf.w_o)
        nets.conv(lf, 2, xd, wts(lf, 7), y, _abi.EPI_RELU)
        done("first layer 7x7/s2", y)
    if only in ("", "tc"):
        for x3 in (False, True):
            for (ci, co, h, f, s, n) in ((64, 128, 18, 3, 1, 1), (64, 64, 9, 3, 1, 4),
                                         (64, 72, 17, 3, 2, 1), (256, 64, 8, 1, 1, 2)):
                lc = nets.Layer("c", ci, co, h, h, f, f, s)
                xc = act(n, ci, h, h, 8)
                wp = nets.prepare_tf32(lc, wts(lc, 9), x3=x3)
                skc = act(n, co, lc.h_o, lc.w_o, 10)
                y = nets.Act(n, co, lc.h_o, lc.w_o)
                nets.conv_tf32(lc, n, xc, wp, y, _abi.EPI_ADD_RELU, skc, x3=x3)
                done(f"{'tf32x3' if x3 else 'tf32'} {ci}->{co} {f}x{f}/s{s} n{n}", y)
    if only in ("", "layout"):
        z = nets.Act(2, 64, 8, 8, halo=1)
        nets.maxpool_into(sk, z)
        done("maxpool", z)
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
