"""Bounds checks of our own (compute-sanitizer is closed on the GPU pool,
profiles/r2_sanitizer_closed.txt): every buffer of a launch sits inside a
larger allocation with guard bands -- NaN around inputs, weights and skip
maps (an out-of-bounds read that reaches a stored output turns it NaN), a
sentinel around the output (an out-of-bounds write changes it).  Each launch
must leave the guards intact and produce results bitwise equal to the same
launch on plain allocations.  Paths: FFMA tiles, forced split-K, tail split,
fused pool, C_o range, first-layer reader, TF32 / split-TF32 (stacked,
strided), max-pool."""
import math
import os

import pytest
import torch

from paper_1809_10170_b200 import _abi, nets

pytestmark = pytest.mark.gpu
GUARD = 1 << 16  # floats per band (256 KB)
SENTINEL = 12345.5


def _guarded(t: torch.Tensor, fill: float):
    big = torch.full((2 * GUARD + t.numel(),), fill, dtype=t.dtype, device=t.device)
    inner = big[GUARD:GUARD + t.numel()].view(t.shape)
    inner.copy_(t)
    return big, inner


def _clone_act(a: nets.Act, fill: float):
    import copy
    b = copy.copy(a)
    big, b.buf = _guarded(a.buf, fill)
    return b, big


def _check_guards(big, n, fill, what):
    lo, hi = big[:GUARD], big[GUARD + n:]
    if math.isnan(fill):
        assert bool(lo.isnan().all() and hi.isnan().all()), f"{what}: input guard written"
    else:
        assert bool((lo == fill).all() and (hi == fill).all()), f"{what}: write outside the view"


def _run_pair(name, make_out, run):
    """run(guarded: bool, out) with inputs taken guarded / plain."""
    y0 = make_out()
    run(False, y0)
    y1, ybig = _clone_act(make_out(), SENTINEL)
    run(True, y1)
    torch.cuda.synchronize()
    _check_guards(ybig, y1.buf.numel(), SENTINEL, name)
    assert bool(torch.isfinite(y1.buf).all()), f"{name}: NaN reached the output (OOB read)"
    assert torch.equal(y0.buf, y1.buf), f"{name}: guarded result differs"


def _act(n, c, h, w, seed, halo=0):
    a = nets.Act(n, c, h, w, halo=halo)
    nets._fill(a.buf, seed, 1)
    return a


def _w(l, seed):
    wd = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), device="cuda")
    nets._fill(wd, seed, 2)
    return nets.pack_weights(wd, l.first)


@pytest.mark.parametrize("ks", [0, 2, 4, 16])
@pytest.mark.parametrize("tv", [1, 2, 3])
def test_ffma_guards(tv, ks, monkeypatch):
    if ks:
        monkeypatch.setenv("DCONV_KSPLIT", str(ks))
    for (ci, co, h, f, s, n) in ((64, 64, 18, 3, 1, 2), (24, 40, 13, 5, 1, 3),
                                 (96, 72, 13, 1, 2, 2), (40, 136, 15, 3, 2, 1)):
        l = nets.Layer("g", ci, co, h, h, f, f, s)
        x, w, sk = _act(n, ci, h, h, 1), _w(l, 2), _act(n, co, l.h_o, l.w_o, 3)
        xg, _ = _clone_act(x, float("nan"))
        skg, _ = _clone_act(sk, float("nan"))
        _, wg = _guarded(w, float("nan"))

        def run(g, y):
            nets.conv(l, n, xg if g else x, wg if g else w, y, _abi.EPI_ADD_RELU,
                      skg if g else sk, tile_variant=tv)
        _run_pair(f"ffma tile {tv} ks {ks} {l}", lambda: nets.Act(n, co, l.h_o, l.w_o, halo=1), run)


def test_ffma_tail_pool_corange_first_guards():
    lt = nets.Layer("t", 64, 64, 10, 10, 3, 3, 1)
    x, w = _act(150, 64, 10, 10, 4), _w(lt, 5)
    xg, _ = _clone_act(x, float("nan"))
    _, wg = _guarded(w, float("nan"))
    _run_pair("tail split", lambda: nets.Act(150, 64, 8, 8),
              lambda g, y: nets.conv(lt, 150, xg if g else x, wg if g else w, y, _abi.EPI_RELU))
    lp = nets.Layer("p", 16, 64, 34, 34, 3, 3, 1)
    x, w = _act(2, 16, 34, 34, 6), _w(lp, 7)
    xg, _ = _clone_act(x, float("nan"))
    _run_pair("fused pool", lambda: nets.Act(2, 64, 16, 16, halo=1),
              lambda g, y: nets.conv(lp, 2, xg if g else x, w, y,
                                     _abi.EPI_RELU | _abi.EPI_MAXPOOL, tile_variant=2))
    lc = nets.Layer("c", 64, 64, 18, 18, 3, 3, 1)
    x, w = _act(1, 64, 18, 18, 8), _w(lc, 9)
    xg, _ = _clone_act(x, float("nan"))
    _run_pair("co range", lambda: nets.Act(1, 64, 16, 16, halo=1),
              lambda g, y: nets.conv(lc, 1, xg if g else x, w, y.block_view(4, 2),
                                     _abi.EPI_RELU, None, None, None, (4, 2)))
    for (f, s, hi) in ((3, 1, 34), (7, 2, 37), (11, 4, 51)):
        lf = nets.Layer("f", 3, 64, hi, hi, f, f, s, first=True)
        xd = torch.empty((2, 3, hi, hi), device="cuda")
        nets._fill(xd, 10, 1)
        _, xdg = _guarded(xd, float("nan"))
        w = _w(lf, 11)
        _run_pair(f"first {f}x{f}/s{s}", lambda: nets.Act(2, 64, lf.h_o, lf.w_o, halo=1),
                  lambda g, y: nets.conv(lf, 2, xdg if g else xd, w, y, _abi.EPI_RELU))


@pytest.mark.parametrize("x3", [False, True])
def test_tensor_core_guards(x3):
    for (ci, co, h, f, s, n) in ((64, 128, 18, 3, 1, 1), (64, 64, 9, 3, 1, 4),
                                 (64, 72, 17, 3, 2, 2), (256, 64, 8, 1, 1, 2),
                                 (128, 256, 9, 3, 1, 8)):
        l = nets.Layer("c", ci, co, h, h, f, f, s)
        x, sk = _act(n, ci, h, h, 12), _act(n, co, l.h_o, l.w_o, 13)
        wp = nets.prepare_tf32(l, _w(l, 14), x3=x3)
        xg, _ = _clone_act(x, float("nan"))
        skg, _ = _clone_act(sk, float("nan"))
        _, wpg = _guarded(wp, float("nan"))
        _run_pair(f"{'tf32x3' if x3 else 'tf32'} {l}", lambda: nets.Act(n, co, l.h_o, l.w_o, halo=1),
                  lambda g, y: nets.conv_tf32(l, n, xg if g else x, wpg if g else wp, y,
                                              _abi.EPI_ADD_RELU, skg if g else sk, x3=x3))


def test_maxpool_guards():
    x = _act(2, 64, 16, 16, 15)
    xg, _ = _clone_act(x, float("nan"))
    _run_pair("maxpool", lambda: nets.Act(2, 64, 8, 8, halo=1),
              lambda g, y: nets.maxpool_into(xg if g else x, y))
