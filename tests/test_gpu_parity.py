"""GPU parity: every CUDA kernel of libdconv_b200.so, called through the
C-ABI, against the CPU oracle (oracle/, pinned to the reference by
tests/test_oracle.py) on identical seeded inputs.

Tolerance (BASELINE.json north_star): fp32 direct conv
|a - b| <= 1e-4 + 1e-5*|b| per element against conv_oracle64
(reference.cpp:70-87); layout repacks, ReLU, skip-add and max-pool bit-exact.
"""
import ctypes
import zlib

import numpy as np
import pytest
import torch

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-4, 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1809_10170_b200._abi as abi
    abi.lib()  # loud failure if the extension is missing
    yield


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def assert_tol(got, want, what=""):
    ok, nbad, err = po.within_tol(got, want, ATOL, RTOL)
    assert ok, f"{what}: {nbad} elements out of tolerance, max abs err {err:.3g}"


# ------------------------------------------------------------------ helpers
from paper_1809_10170_b200 import dconv as D  # noqa: E402
from paper_1809_10170_b200 import _abi, nets  # noqa: E402


def run_conv(x, k, s, c_ib, c_ob, algo=_abi.ALGO_AUTO, relu=False, skip=None, tile_variant=0):
    """dense numpy x [c][h][w], k [ci][co][hf][wf] -> blocked numpy output."""
    ci, hi, wi = x.shape
    _, co, hf, wf = k.shape
    shape = D.ConvShape(ci, co, hi, wi, hf, wf, s)
    xb = D.BlockedFeatureMap(ci, hi, wi, c_ib, data=dev(po.pack_feature_map(x, c_ib)[None]))
    kb = D.BlockedKernel(ci, co, hf, wf, c_ob, c_ib, data=dev(po.pack_kernel(k, c_ob, c_ib)))
    sk = None
    if skip is not None:
        sk = D.BlockedFeatureMap(co, shape.h_o, shape.w_o, c_ob, data=dev(skip[None]))
    y = D.conv_direct(xb, kb, shape, D.BlockingParams(c_ob, 1, c_ib), relu=relu, skip=sk,
                      algo=algo, tile_variant=tile_variant)
    return host(y.data)[0]


# ------------------------------------------------------------------ cases
def test_cfg1_full_parity():
    """BASELINE cfg1: 64->64 3x3 s1 58->56, b1, fp32, FFMA path."""
    x = po.uniform((64, 58, 58), 1809, 0)
    k = po.uniform((64, 64, 3, 3), 1809, 1)
    got = run_conv(x, k, 1, 8, 8, algo=_abi.ALGO_FFMA)
    want = po.pack_feature_map(po.conv_oracle64(x, k, 1), 8)
    assert_tol(got, want, "cfg1")


def test_golden_fixtures_generic_and_ffma():
    """Reference-generated golden vectors (tests/golden) through both paths."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    names = sorted({k.split("/")[0] for k in g.files})
    for n in names:
        ci, co, hi, wi, hf, wf, s, cib, cob = g[f"{n}/geom"].tolist()
        x, k = g[f"{n}/x"], g[f"{n}/k"]
        got = run_conv(x, k, s, cib, cob, algo=_abi.ALGO_GENERIC)
        assert_tol(got, g[f"{n}/y_oracle64_blocked"], f"{n}/generic")
        got8 = run_conv(x, k, s, 8, 8, algo=_abi.ALGO_FFMA)
        assert_tol(got8, po.pack_feature_map(g[f"{n}/y_oracle64"], 8), f"{n}/ffma")


def test_spec_trivial_direct():
    """1x1x1 [2]*[3] -> 6, both kernels."""
    x = np.array([[[2.0]]], np.float32)
    k = np.array([[[[3.0]]]], np.float32)
    assert run_conv(x, k, 1, 1, 1, algo=_abi.ALGO_GENERIC).ravel()[0] == 6.0
    y = run_conv(x, k, 1, 8, 8, algo=_abi.ALGO_FFMA).ravel()
    assert y[0] == 6.0 and not y[1:].any()


def test_acceptance1_random_shapes():
    """SPEC.md:615 property suite (seeded, channels <= 64, spatial <= 32,
    filters {1,3,5,7,11}, strides {1,2,4}) on the FFMA kernel."""
    rng = np.random.default_rng(1809)
    for t in range(120):
        hf = int(rng.choice([1, 3, 5, 7, 11]))
        wf = hf
        s = int(rng.choice([1, 2, 4]))
        ci, co = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        ho_max = (32 - hf) // s + 1
        if ho_max < 1:
            continue
        ho, wo = int(rng.integers(1, ho_max + 1)), int(rng.integers(1, ho_max + 1))
        hi, wi = (ho - 1) * s + hf, (wo - 1) * s + wf
        x = po.uniform((ci, hi, wi), 2000 + t, 0)
        k = po.uniform((ci, co, hf, wf), 2000 + t, 1)
        want = po.pack_feature_map(po.conv_oracle64(x, k, s), 8)
        assert_tol(run_conv(x, k, s, 8, 8, algo=_abi.ALGO_FFMA), want,
                   f"case {t} ({ci},{co},{hi},{wi},{hf},{s})")


def test_generic_any_block_sizes():
    """Every (c_ob, c_ib) of the reference API has a CUDA path."""
    rng = np.random.default_rng(5)
    for t, (cob, cib) in enumerate([(1, 1), (4, 2), (8, 4), (3, 5), (16, 16), (32, 8), (6, 8)]):
        ci, co = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        x = po.uniform((ci, 9, 11), 300 + t, 0)
        k = po.uniform((ci, co, 3, 3), 300 + t, 1)
        want = po.pack_feature_map(po.conv_oracle64(x, k, 2), cob)
        assert_tol(run_conv(x, k, 2, cib, cob, algo=_abi.ALGO_GENERIC), want, f"{cob},{cib}")


def test_edge_tiles_spec():
    """w_o = 7 (ragged tiles), c_o = 6 (padded block)."""
    x = po.uniform((5, 9, 9), 77, 0)
    k = po.uniform((5, 6, 3, 3), 77, 1)
    y = run_conv(x, k, 1, 8, 8, algo=_abi.ALGO_FFMA)
    assert_tol(y, po.pack_feature_map(po.conv_oracle64(x, k, 1), 8), "edge")
    assert not y[..., 6:].any(), "padded output channels must be exact 0"


def test_fused_epilogues():
    x = po.uniform((24, 12, 12), 88, 0)
    k = po.uniform((24, 16, 3, 3), 88, 1)
    ref = po.pack_feature_map(po.conv_oracle64(x, k, 1), 8)
    skip = po.pack_feature_map(po.uniform((16, 10, 10), 88, 2), 8)
    assert_tol(run_conv(x, k, 1, 8, 8, relu=True), np.maximum(ref, 0), "relu")
    assert_tol(run_conv(x, k, 1, 8, 8, skip=skip), ref + skip, "add")
    assert_tol(run_conv(x, k, 1, 8, 8, relu=True, skip=skip), np.maximum(ref + skip, 0),
               "add_relu")
    for algo in (_abi.ALGO_GENERIC,):
        assert_tol(run_conv(x, k, 1, 8, 8, algo=algo, relu=True, skip=skip),
                   np.maximum(ref + skip, 0), "generic add_relu")


def test_determinism_bitwise():
    """repeated runs are bitwise identical (no atomics)."""
    x = po.uniform((64, 30, 30), 9, 0)
    k = po.uniform((64, 128, 3, 3), 9, 1)
    a = run_conv(x, k, 1, 8, 8)
    b = run_conv(x, k, 1, 8, 8)
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ layouts
@pytest.mark.parametrize("cob,cib", [(1, 1), (4, 2), (8, 4), (8, 8), (3, 5), (8, 3), (32, 32)])
def test_pack_kernel_bitexact(cob, cib):
    k = po.uniform((13, 21, 3, 3), 50, cob * 7 + cib)
    got = D.pack_kernel(dev(k), cob, cib)
    assert np.array_equal(host(got.data), po.pack_kernel(k, cob, cib))
    assert np.array_equal(host(D.unpack_kernel(got)), k)


@pytest.mark.parametrize("cb", [1, 2, 3, 8, 16])
def test_pack_feature_map_bitexact(cb):
    x = po.uniform((2, 11, 7, 9), 60, cb)
    got = D.pack_feature_map(dev(x), cb)
    want = np.stack([po.pack_feature_map(x[i], cb) for i in range(2)])
    assert np.array_equal(host(got.data), want)
    assert np.array_equal(host(D.unpack_feature_map(got)), x)


def test_pack_feature_map_halo():
    import ctypes
    x = po.uniform((1, 5, 4, 6), 61, 0)
    out = torch.full((1, 1, 6, 8, 8), 7.0, device="cuda")
    _abi.check(_abi.lib().dconv_cuda_pack_feature_map(_abi.ptr(dev(x)), 1, 5, 4, 6, 8, 1,
                                                     _abi.ptr(out), _abi.stream_ptr()))
    o = host(out)
    want = np.zeros((1, 1, 6, 8, 8), np.float32)
    want[0, :, 1:5, 1:7, :] = po.pack_feature_map(x[0], 8)
    assert np.array_equal(o, want)


def test_layout_counter_and_chain():
    """chain of 1x1 weights 2.0 then 3.0 on 1.0 -> 6.0; no
    layout transforms inside; c_ib/c_ob mismatch -> layout error."""
    x = D.pack_feature_map(dev(np.ones((1, 1, 1), np.float32)), 8)
    k1 = D.pack_kernel(dev(np.full((1, 1, 1, 1), 2.0, np.float32)), 8, 8)
    k2 = D.pack_kernel(dev(np.full((1, 1, 1, 1), 3.0, np.float32)), 8, 8)
    sh = D.ConvShape(1, 1, 1, 1, 1, 1, 1)
    p = D.BlockingParams(8, 1, 8)
    before = D.layout_transform_count()
    y = D.layer_chain(x, [(k1, sh, p), (k2, sh, p)])
    assert D.layout_transform_count() == before
    assert host(y.data).ravel()[0] == 6.0
    k3 = D.pack_kernel(dev(np.ones((1, 1, 1, 1), np.float32)), 4, 4)
    with pytest.raises(ValueError, match="layout"):
        D.layer_chain(x, [(k1, sh, p), (k3, sh, D.BlockingParams(4, 1, 4))])


def test_shape_errors_match_reference():
    with pytest.raises(ValueError, match="ConvShape"):
        D.ConvShape(3, 64, 230, 230, 7, 7, 2)
    with pytest.raises(ValueError, match="ConvShape"):
        D.ConvShape(1, 1, 2, 2, 3, 3)


# ------------------------------------------------------------ element-wise
def test_relu_add_maxpool_bitexact():
    a = po.uniform((3, 2, 6, 10, 8), 70, 0)
    b = po.uniform((3, 2, 6, 10, 8), 70, 1)
    ta, tb = dev(a), dev(b)
    A = D.BlockedFeatureMap(16, 6, 10, 8, n=3, data=ta.clone())
    B = D.BlockedFeatureMap(16, 6, 10, 8, n=3, data=tb)
    assert np.array_equal(host(D.add_blocked(A, B).data), a + b)
    assert np.array_equal(host(D.add_blocked(A, B, relu=True).data), np.maximum(a + b, 0))
    assert np.array_equal(host(D.maxpool2x2_blocked(A).data),
                          a.reshape(3, 2, 3, 2, 5, 2, 8).max(axis=(3, 5)))
    D.relu_blocked(A)
    assert np.array_equal(host(A.data), np.maximum(a, 0))
    x = dev(np.array([-1.0, 0.0, 2.0], np.float32))
    _abi.check(_abi.lib().dconv_cuda_relu_blocked(_abi.ptr(x), 3, _abi.stream_ptr()))
    assert host(x).tolist() == [0.0, 0.0, 2.0]


# ------------------------------------------------------- views and sharding
def test_output_into_halo_and_crop_view():
    """Producer writes into the interior of a halo'd consumer buffer; a
    consumer reads a crop (ResNet stride-2 projection 55x55 of 56x56)."""
    n = 2
    x = po.uniform((n, 16, 12, 12), 90, 0)
    k = po.uniform((16, 24, 1, 1), 90, 1)
    a = nets.Act(n, 16, 12, 12)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    l = nets.Layer("proj", 16, 24, 11, 11, 1, 1, 2)
    y = nets.Act(n, 24, 6, 6, halo=1)
    nets.conv(l, n, a, nets.pack_weights(dev(k), False), y)
    got = host(y.buf)
    for i in range(n):
        want = po.pack_feature_map(po.conv_oracle64(x[i, :, :11, :11], k, 2), 8)
        assert_tol(got[i, :, 1:7, 1:7, :], want, "crop->halo")
    ring = got.copy()
    ring[:, :, 1:7, 1:7, :] = 0
    assert not ring.any(), "halo ring must stay zero"


def test_co_block_sharding_ranges():
    """C_o-block sharding: each rank computes a contiguous j' range into its
    own slice buffer; the concatenation equals the full conv (bitwise)."""
    import ctypes
    x = po.uniform((32, 14, 14), 95, 0)
    k = po.uniform((32, 64, 3, 3), 95, 1)
    xb = dev(po.pack_feature_map(x, 8)[None])
    kb = dev(po.pack_kernel(k, 8, 8))
    full = run_conv(x, k, 1, 8, 8)
    parts = []
    for r in range(4):
        d = D.make_desc(D.ConvShape(32, 64, 14, 14, 3, 3, 1), 1, 8, 8)
        d.co_block_begin, d.co_block_count = 2 * r, 2
        out = torch.empty((1, 2, 12, 12, 8), device="cuda")
        _abi.check(_abi.lib().dconv_cuda_conv_direct(ctypes.byref(d), _abi.ptr(xb),
                                                     _abi.ptr(kb), 0, _abi.ptr(out),
                                                     _abi.stream_ptr()))
        parts.append(host(out)[0])
    assert np.array_equal(np.concatenate(parts, 0), full)


# --------------------------------------------------- BASELINE config layers
def _rows(h):
    return sorted({0, 1, h // 2, h - 2, h - 1} & set(range(h)))


ALL_LAYERS = [(cfg, l) for cfg in ("cfg1", "alexnet", "vgg16", "googlenet") for l in
              nets.CONFIGS[cfg]] + [("resnet50", l) for l in {
                  (l.c_i, l.c_o, l.h_i, l.h_f, l.s): l for l in nets.CONFIGS["resnet50"]}.values()]


@pytest.mark.parametrize("cfg,layer", ALL_LAYERS, ids=[f"{c}-{l.name}" for c, l in ALL_LAYERS])
def test_config_layer_parity(cfg, layer):
    """Every distinct layer shape of BASELINE.json configs 1-5 at batch 2,
    fp32, vs conv_oracle64 on sampled output rows (edges + middle) of both
    images."""
    l, n = layer, 2
    sid = zlib.crc32(f"{cfg}/{l.name}".encode()) % 10_000
    k = po.uniform((l.c_i, l.c_o, l.h_f, l.w_f), 4000 + sid, 1)
    w = nets.pack_weights(dev(k), l.first)
    assert np.array_equal(host(w), po.pack_kernel(k, 8, l.c_i if l.first else 8))
    xs = [po.uniform((l.c_i, l.h_i, l.w_i), 4000 + sid, 10 + i) for i in range(n)]
    y = nets.Act(n, l.c_o, l.h_o, l.w_o)
    if l.first:
        nets.conv(l, n, dev(np.stack(xs)), w, y)
    else:
        a = nets.Act(n, l.c_i, l.h_i, l.w_i)
        a.buf.copy_(dev(np.stack([po.pack_feature_map(xx, 8) for xx in xs])))
        nets.conv(l, n, a, w, y)
    got = host(y.buf)
    rows = _rows(l.h_o)
    kb = po.pack_kernel(k, 8, 8)
    for i in range(n):
        xb = po.pack_feature_map(xs[i], 8)
        for r in rows:
            want = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, r, r + 1)
            assert_tol(got[i, :, r], want[:, r], f"{cfg}/{l.name} img {i} row {r}")


@pytest.mark.parametrize("s,f,ci,co", [(1, 3, 3, 64), (2, 7, 3, 64), (4, 11, 3, 96), (1, 5, 3, 20),
                                       (1, 1, 4, 8), (2, 3, 1, 64), (3, 3, 3, 16), (1, 3, 3, 72)])
def test_first_layer_reader_variants(s, f, ci, co):
    """Dense-input first layer (all specialisations + the generic fallback
    for (s=3, f=3)) vs conv_oracle64, batch 2, ragged tiles, relu epilogue."""
    n = 2
    ho, wo = 13, 21
    hi, wi = (ho - 1) * s + f, (wo - 1) * s + f
    x = po.uniform((n, ci, hi, wi), 5000 + s * 100 + f, 0)
    k = po.uniform((ci, co, f, f), 5000 + s * 100 + f, 1)
    l = nets.Layer("first", ci, co, hi, wi, f, f, s, first=True)
    y = nets.Act(n, co, ho, wo)
    nets.conv(l, n, dev(x), nets.pack_weights(dev(k), True), y, epilogue=_abi.EPI_RELU)
    got = host(y.buf)
    for i in range(n):
        want = np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, s), 8), 0)
        assert_tol(got[i], want, f"first s={s} f={f} img {i}")


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_ffma_tile_variants(variant):
    """The FFMA CTA tiles (128 px x 128 ch, 256 px x 64 ch, 128 px x 64 ch, 256 px x 32 ch) on ragged shapes,
    strides, filter widths 1/3/5/7 (templated and runtime), and a K = 4608
    layer where the TMEM two-level sum matters (desc.tile_variant)."""
    cases = [(64, 64, 58, 58, 3, 1), (24, 40, 17, 23, 5, 1), (16, 136, 19, 21, 7, 2),
             (96, 72, 13, 31, 1, 2), (512, 128, 16, 16, 3, 1), (200, 16, 9, 9, 3, 2)]
    for t, (ci, co, hi, wi, f, s) in enumerate(cases):
        x = po.uniform((ci, hi, wi), 7000 + t, variant)
        k = po.uniform((ci, co, f, f), 7000 + t, 10 + variant)
        want = po.pack_feature_map(po.conv_oracle64(x, k, s), 8)
        assert_tol(run_conv(x, k, s, 8, 8, algo=_abi.ALGO_FFMA, tile_variant=variant + 1), want,
                   f"variant {variant} case {t}")


@pytest.mark.parametrize("ks", [0, 1, 2, 4])
def test_ffma_32_channel_tile_epilogues(ks, monkeypatch):
    """The 256 px x 32 ch CTA tile (8 x 4 warp shape, lanes 4-7 of a
    quarter-warp reading the channel halves swapped): GoogLeNet's 5x5 16->32
    and 3x3 112->224 (seven 32-channel groups) shapes and a ragged C_o, with
    the fused skip-add + ReLU epilogue (epilogue warpgroup) and forced split-K
    factors (DSMEM reduction) -- every image against the oracle."""
    if ks:
        monkeypatch.setenv("DCONV_KSPLIT", str(ks))
    cases = [(16, 32, 12, 12, 5, 1, 3), (112, 224, 9, 9, 3, 1, 2), (40, 20, 11, 13, 3, 2, 2),
             (64, 96, 8, 8, 1, 1, 3)]
    for t, (ci, co, hi, wi, f, s, n) in enumerate(cases):
        l = nets.Layer("t32", ci, co, hi, wi, f, f, s)
        x = po.uniform((n, ci, hi, wi), 1200 + t, ks)
        k = po.uniform((ci, co, f, f), 1210 + t, ks)
        sk = po.uniform((n, co, l.h_o, l.w_o), 1220 + t, ks)
        a = nets.Act(n, ci, hi, wi)
        a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
        skip = nets.Act(n, co, l.h_o, l.w_o)
        skip.buf.copy_(dev(np.stack([po.pack_feature_map(sk[i], 8) for i in range(n)])))
        y = nets.Act(n, co, l.h_o, l.w_o)
        nets.conv(l, n, a, nets.pack_weights(dev(k), False), y, _abi.EPI_ADD | _abi.EPI_RELU,
                  skip, tile_variant=4)
        got = host(y.buf)
        for i in range(n):
            want = np.maximum(po.conv_oracle64(x[i], k, s) + sk[i], 0)
            assert_tol(got[i], po.pack_feature_map(want, 8), f"ks {ks} case {t} img {i}")


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_batched_stacked_tiles(variant):
    """Pixel tiles over the batch-stacked output span several images (maps of
    height 1..9 with tiles of up to 64 rows): every image checked."""
    rng = np.random.default_rng(900 + variant)
    for t in range(14):
        n = int(rng.integers(2, 7))
        f = int(rng.choice([1, 3, 5]))
        s = int(rng.choice([1, 2]))
        ho, wo = int(rng.integers(1, 10)), int(rng.integers(1, 16))
        ci, co = int(rng.integers(1, 40)), int(rng.integers(1, 150))
        hi, wi = (ho - 1) * s + f, (wo - 1) * s + f
        x = po.uniform((n, ci, hi, wi), 950 + t, variant)
        k = po.uniform((ci, co, f, f), 960 + t, variant)
        l = nets.Layer("b", ci, co, hi, wi, f, f, s)
        a = nets.Act(n, ci, hi, wi)
        a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
        y = nets.Act(n, co, ho, wo)
        nets.conv(l, n, a, nets.pack_weights(dev(k), False), y, tile_variant=variant + 1)
        got = host(y.buf)
        for i in range(n):
            want = po.pack_feature_map(po.conv_oracle64(x[i], k, s), 8)
            assert_tol(got[i], want, f"v{variant} case {t} img {i} ({n},{ci},{co},{hi},{wi},{f},{s})")


# ------------------------------------------------ chains (wiring, teacher-forced)
def _conv_io(plan):
    """(layer, input Act/tensor, output Act, epilogue, skip) per conv, recorded
    by re-wrapping nets.conv during a plan run."""
    rec = []
    orig = nets.conv

    def spy(l, n, x, w, out, epilogue=0, skip=None, stream=None, in_view=None, co_range=None,
            **kw):
        orig(l, n, x, w, out, epilogue, skip, stream, in_view, co_range, **kw)
        torch.cuda.synchronize()
        xin = x.clone() if isinstance(x, torch.Tensor) else x.buf.clone()
        rec.append((l, xin, out.buf.clone(), out, epilogue, skip.buf.clone() if skip else None,
                    skip, w))
    nets.conv = spy
    try:
        plan.run()
    finally:
        nets.conv = orig
    return rec


@pytest.mark.parametrize("config", ["vgg16", "resnet50", "alexnet", "googlenet"])
def test_chain_wiring_teacher_forced(config):
    plan = nets.build_plan(config, 1)
    rec = _conv_io(plan)
    assert len(rec) == len(plan.layers)
    for l, xin, yout, out, epi, skb, skip, w in rec:
        xin = xin.cpu().numpy()[0]
        got = yout.cpu().numpy()[0]
        if l.first:
            # dense input -> blocked c_b = 8 (zero channel padding is exact)
            xb = po.pack_feature_map(np.ascontiguousarray(xin[:, :l.h_i, :l.w_i]), 8)
        else:
            xb = np.ascontiguousarray(xin[:, :l.h_i, :l.w_i, :])  # crop views (projections)
        kd = po.unpack_kernel(w.cpu().numpy(), l.c_i, l.c_o) if not l.first else None
        kb = po.pack_kernel(kd, 8, 8) if kd is not None else po.pack_kernel(
            _first_dense(w.cpu().numpy(), l), 8, 8)
        h = out.halo
        if epi & _abi.EPI_MAXPOOL:  # fused 2x2/s2 pool: compare pooled rows
            hp, wp = l.h_o // 2, l.w_o // 2
            for rp in sorted({0, hp // 2, hp - 1}):
                two = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, 2 * rp, 2 * rp + 2)
                two = two[:, 2 * rp:2 * rp + 2]
                if epi & _abi.EPI_RELU:
                    two = np.maximum(two, 0)
                want = two.reshape(two.shape[0], 2, wp, 2, 8).max(axis=(1, 3))
                g = got[:, h + rp, h:h + wp, :]
                scale = max(1.0, float(np.abs(want).max()))
                err = float(np.abs(g - want).max())
                assert err <= 1e-5 * scale + 1e-4, f"{config}/{l.name} pooled row {rp}: err {err}"
            continue
        for r in sorted({0, l.h_o // 2, l.h_o - 1}):
            want = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, r, r + 1)[:, r]
            if epi & _abi.EPI_ADD:
                sk = skb.cpu().numpy()[0]
                want = want + sk[:, skip.halo + r, skip.halo:skip.halo + l.w_o, :]
            if epi & _abi.EPI_RELU:
                want = np.maximum(want, 0)
            g = got[:, h + r, h:h + l.w_o, :]
            scale = max(1.0, float(np.abs(want).max()))
            err = float(np.abs(g - want).max())
            assert err <= 1e-5 * scale + 1e-4, f"{config}/{l.name} row {r}: err {err} scale {scale}"


def _first_dense(wb, l):
    """blocked first-layer weights (c_ib = c_i) -> dense [c_i][c_o][h_f][w_f]"""
    return po.unpack_kernel(wb, l.c_i, l.c_o)


def test_co_shard_plan_world1_matches_unsharded():
    """The C_o-sharded plan (slices + all-gather via a real 1-rank NCCL group)
    reproduces the unsharded plan bitwise on ResNet-50 b1."""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a = nets.build_plan("resnet50", 1, seed=5)
        b = nets.build_plan("resnet50", 1, seed=5, shard=(0, 1, None))
        a.run()
        b.run()
        torch.cuda.synchronize()
        assert any(s.kind == "gather" for s in b.steps)
        assert torch.equal(a.output.buf, b.output.buf)
        # on a side stream (as bench.py runs plans): the all-gathers must be
        # ordered after the convs on that stream, not on torch's current one
        b.output.buf.zero_()
        side = torch.cuda.Stream()
        for _ in range(3):
            b.run(side)
        side.synchronize()
        assert torch.equal(a.output.buf, b.output.buf)
    finally:
        dist.destroy_process_group()


def test_peer_store_epilogue_writes_every_copy():
    """The fused C_o-shard gather kernel path: a rank's output blocks are
    stored into its own map and, at the same offsets, into every peer copy
    (here local buffers stand in for the P2P-mapped peers); blocks owned by
    other ranks are left untouched in all copies.  FFMA and first-layer
    reader, ReLU and ADD_RELU epilogues."""
    import ctypes
    lib = _abi.lib()
    # blocked 3x3 layer: rank 1 of 2 computes output blocks [2, 4) of 4
    ci, co, h = 16, 32, 12
    x = po.uniform((ci, h, h), 9500, 0)
    k = po.uniform((ci, co, 3, 3), 9500, 1)
    skip = po.pack_feature_map(po.uniform((co, h - 2, h - 2), 9500, 2), 8)
    l = nets.Layer("pe", ci, co, h, h, 3, 3, 1)
    a = nets.Act(1, ci, h, h)
    a.buf.copy_(dev(po.pack_feature_map(x, 8)[None]))
    sk = nets.Act(1, co, h - 2, h - 2)
    sk.buf.copy_(dev(skip[None]))
    copies = [nets.Act(1, co, h - 2, h - 2, halo=1) for _ in range(3)]
    for c in copies:
        c.buf.fill_(7.0)
    b0, cnt = 2, 2
    peers = [c.base() + 4 * b0 * c.blk for c in copies[1:]]
    nets.conv(l, 1, a, nets.pack_weights(dev(k), False), copies[0].block_view(b0),
              _abi.EPI_ADD_RELU, sk, co_range=(b0, cnt), peers=peers)
    want = np.maximum(po.pack_feature_map(po.conv_oracle64(x, k, 1), 8) + skip, 0)
    ref = host(copies[0].buf)
    for c in copies:
        got = host(c.buf)
        assert np.array_equal(got, ref), "peer copy differs from the local store"
        assert_tol(got[0, b0:b0 + cnt, 1:-1, 1:-1], want[b0:b0 + cnt], "peer-store conv")
        assert (got[0, :b0] == 7.0).all() and (got[0, :, 0] == 7.0).all()
    # first-layer reader with peers
    xf = po.uniform((3, 23, 23), 9501, 0)
    kf = po.uniform((3, 64, 7, 7), 9501, 1)
    lf = nets.Layer("pf", 3, 64, 23, 23, 7, 7, 2, True)
    outs = [nets.Act(1, 64, lf.h_o, lf.w_o) for _ in range(2)]
    nets.conv(lf, 1, dev(xf[None]), nets.pack_weights(dev(kf), True), outs[0].block_view(4),
              _abi.EPI_RELU, co_range=(4, 4), peers=[outs[1].base() + 4 * 4 * outs[1].blk])
    wantf = np.maximum(po.pack_feature_map(po.conv_oracle64(xf, kf, 2), 8), 0)
    g0, g1 = host(outs[0].buf), host(outs[1].buf)
    assert np.array_equal(g0, g1)
    assert_tol(g0[0, 4:], wantf[4:], "peer-store first layer")
    assert not g0[0, :4].any()
    # argument checks
    d = nets._desc(l, 1)
    bad = (ctypes.c_void_p * 8)(*([peers[0]] * 8))
    with pytest.raises(ValueError, match="n_peers"):
        _abi.check(lib.dconv_cuda_conv_direct_peers(ctypes.byref(d), a.base(), 0, 0,
                                                    copies[0].base(), bad, 8, 0))


def test_co_shard_peer_gather_plan_world1():
    """The symmetric-memory ("peer") C_o-shard plan on a 1-rank NCCL group:
    symmetric buffers, block views, device barriers -- bitwise equal to the
    unsharded plan on ResNet-50 b1 and VGG-16 b1."""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29519")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        for cfg in ("resnet50", "vgg16"):
            a = nets.build_plan(cfg, 1, seed=6)
            b = nets.build_plan(cfg, 1, seed=6, shard=(0, 1, None), gather_mode="peer")
            assert any(s.kind == "barrier" for s in b.steps)
            assert not any(s.kind == "gather" for s in b.steps)
            for _ in range(2):  # repeated steps reuse the symmetric buffers
                a.run()
                b.run()
            torch.cuda.synchronize()
            assert torch.equal(a.output.buf, b.output.buf), cfg
    finally:
        dist.destroy_process_group()


def test_cluster_slots_cached_per_kernel():
    """The launcher caches co-resident cluster counts per (device, kernel
    instantiation, ks): driving all three CTA tiles in one process gives each
    its own answer, equal to a fresh occupancy query of that kernel; then a
    batch-1 split-K layer runs correctly on each tile in turn."""
    lib = _abi.lib()
    for ks in (2, 4, 8, 16):
        for variant in (1, 2, 3, 4, 1):
            cached, fresh = ctypes.c_int(0), ctypes.c_int(0)
            _abi.check(lib.dconv_cuda_ffma_cluster_slots(variant, ks, ctypes.byref(cached),
                                                         ctypes.byref(fresh)))
            assert cached.value == fresh.value, (variant, ks, cached.value, fresh.value)
    x = po.uniform((64, 30, 30), 4242, 0)
    k = po.uniform((64, 64, 3, 3), 4242, 1)
    want = po.pack_feature_map(po.conv_oracle64(x, k, 1), 8)
    for variant in (1, 2, 3, 2):
        assert_tol(run_conv(x, k, 1, 8, 8, algo=_abi.ALGO_FFMA, tile_variant=variant), want,
                   f"tile {variant}")


@pytest.mark.parametrize("ks", [2, 3, 4, 6, 8, 12, 16])
def test_cluster_split_k(ks, monkeypatch):
    """Split-K over a thread-block cluster with the DSMEM reduction, forced
    to ks CTAs per unit: several units per cluster (barrier phases), ragged
    stage splits, every CTA tile; bitwise repeatable."""
    monkeypatch.setenv("DCONV_KSPLIT", str(ks))
    cases = [(64, 64, 58, 58, 3, 1, 1), (40, 136, 17, 23, 3, 1, 3), (96, 72, 13, 31, 1, 2, 2),
             (200, 24, 9, 9, 3, 2, 4), (24, 40, 17, 23, 5, 1, 2), (512, 128, 9, 9, 3, 1, 2)]
    for variant in (0, 1, 2):
        for t, (ci, co, hi, wi, f, s, n) in enumerate(cases):
            x = po.uniform((n, ci, hi, wi), 8000 + t, ks)
            k = po.uniform((ci, co, f, f), 8100 + t, ks)
            l = nets.Layer("k", ci, co, hi, wi, f, f, s)
            a = nets.Act(n, ci, hi, wi)
            a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
            wb = nets.pack_weights(dev(k), False)
            y = nets.Act(n, co, l.h_o, l.w_o)
            nets.conv(l, n, a, wb, y, epilogue=_abi.EPI_RELU, tile_variant=variant + 1)
            got = host(y.buf)
            y2 = nets.Act(n, co, l.h_o, l.w_o)
            nets.conv(l, n, a, wb, y2, epilogue=_abi.EPI_RELU, tile_variant=variant + 1)
            assert np.array_equal(got, host(y2.buf)), "split-K not bitwise repeatable"
            for i in range(n):
                want = np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, s), 8), 0)
                assert_tol(got[i], want, f"ks={ks} v{variant} case {t} img {i}")


# ---------------------------------------------------------- TF32 tensor cores
def run_conv_tf32(x, k, relu=False, skip=None, x3=False):
    """tcgen05/TMEM TF32 path through the C-ABI (stride 1, c_b = 8); ``x3``:
    the split-TF32 entry points."""
    import ctypes
    ci, hi, wi = x.shape[-3:]
    n = x.shape[0] if x.ndim == 4 else 1
    xs = x if x.ndim == 4 else x[None]
    _, co, hf, wf = k.shape
    shape = D.ConvShape(ci, co, hi, wi, hf, wf, 1)
    d = D.make_desc(shape, n, 8, 8, (_abi.EPI_RELU if relu else 0) | (_abi.EPI_ADD if skip is not None else 0))
    xb = dev(np.stack([po.pack_feature_map(xs[i], 8) for i in range(n)]))
    kb = dev(po.pack_kernel(k, 8, 8))
    sz = ctypes.c_int64(0)
    L = _abi.lib()
    sfx = "tf32x3" if x3 else "tf32"
    _abi.check(getattr(L, f"dconv_cuda_{sfx}_prepared_size")(ctypes.byref(d), ctypes.byref(sz)))
    wp = torch.empty(sz.value, device="cuda")
    _abi.check(getattr(L, f"dconv_cuda_prepare_{sfx}_weights")(ctypes.byref(d), _abi.ptr(kb),
                                                               _abi.ptr(wp), _abi.stream_ptr()))
    out = torch.empty((n, (co + 7) // 8, shape.h_o, shape.w_o, 8), device="cuda")
    sk = dev(skip) if skip is not None else None
    _abi.check(getattr(L, f"dconv_cuda_conv_direct_{sfx}")(ctypes.byref(d), _abi.ptr(xb), _abi.ptr(wp),
                                                           _abi.ptr(sk), _abi.ptr(out),
                                                           _abi.stream_ptr()))
    return host(out)


def tf32_bound(x, k):
    """|a - b| <= 2^-9 * sum|x||w| + 1e-5: TF32 keeps 10 of fp32's 23
    mantissa bits (relative error <= 2^-10 per operand, <= 2^-9 per product)."""
    return 2.0 ** -9 * po.pack_feature_map(po.conv_oracle64(np.abs(x), np.abs(k), 1), 8) + 1e-5


@pytest.mark.parametrize("ci,co,h,w,f,n", [(64, 64, 18, 18, 3, 1), (16, 128, 20, 13, 3, 2),
                                            (24, 40, 70, 21, 3, 1), (32, 256, 10, 10, 1, 3),
                                            (8, 72, 12, 12, 5, 1), (96, 136, 9, 30, 3, 2),
                                            (40, 264, 20, 11, 3, 2), (24, 512, 35, 9, 3, 1)])
def test_tf32_tensor_core_parity(ci, co, h, w, f, n):
    x = po.uniform((n, ci, h, w), 9100 + ci, co)
    k = po.uniform((ci, co, f, f), 9200 + ci, co)
    got = run_conv_tf32(x, k)
    for i in range(n):
        want = po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8)
        err = np.abs(got[i].astype(np.float64) - want)
        bound = tf32_bound(x[i], k)
        assert (err <= bound).all(), f"TF32 error {err.max()} exceeds bound (max ratio {(err / bound).max()})"
        assert err.max() > 0 or ci * f * f <= 8  # it really is TF32, not an fp32 fallback


# ---------------------------------------------- split-TF32 (fp32 tolerance)
@pytest.mark.parametrize("ci,co,h,w,f,n", [(64, 64, 18, 18, 3, 1), (16, 128, 20, 13, 3, 2),
                                            (24, 40, 70, 21, 3, 1), (32, 256, 10, 10, 1, 3),
                                            (8, 72, 12, 12, 5, 1), (96, 136, 9, 30, 3, 2),
                                            (40, 264, 20, 11, 3, 2), (24, 512, 35, 9, 3, 1),
                                            (512, 512, 9, 9, 3, 2), (256, 256, 16, 16, 3, 2),
                                            (1024, 256, 14, 14, 1, 2), (64, 64, 58, 58, 3, 1),
                                            (64, 128, 9, 9, 3, 3), (96, 256, 7, 7, 1, 5),
                                            (40, 72, 6, 11, 1, 4)])
def test_tf32x3_meets_fp32_tolerance(ci, co, h, w, f, n):
    """The split-TF32 tensor-core kernel against the fp64 oracle with the
    fp32 FFMA tolerance |a-b| <= 1e-4 + 1e-5|b| (north_star), up to
    K = C_i*H_f*W_f = 4608 (the chunked two-level summation)."""
    x = po.uniform((n, ci, h, w), 9100 + ci, co)
    k = po.uniform((ci, co, f, f), 9200 + ci, co)
    got = run_conv_tf32(x, k, x3=True)
    one = run_conv_tf32(x[:1], k) if ci * f * f > 8 else None
    for i in range(n):
        want = po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8)
        assert_tol(got[i], want, f"tf32x3 img {i}")
        # and with a margin: the chunked sum keeps the worst element at
        # <= 0.52 of the bound (profiles/r1_tf32x3_kernel_accuracy.txt)
        ok, nbad, err = po.within_tol(got[i], want, 0.75 * ATOL, 0.75 * RTOL)
        assert ok, f"tf32x3 img {i}: {nbad} elements beyond 0.75 of the tolerance ({err:.3g})"
    if one is not None:  # the single-pass TF32 kernel does not meet it: x3 is doing work
        want = po.pack_feature_map(po.conv_oracle64(x[0], k, 1), 8)
        assert not po.within_tol(one[0], want, ATOL, RTOL)[0]


@pytest.mark.parametrize("n,h", [(2, 12), (3, 9)])
def test_tf32x3_epilogue_and_padding(n, h):
    """ReLU + skip epilogue and zero padded channels; h = 9 (7x7 output)
    runs with two images stacked per M-tile (the last unit half empty)."""
    x = po.uniform((n, 40, h, h), 95, 0)
    k = po.uniform((40, 20, 3, 3), 95, 1)
    skip = np.stack([po.pack_feature_map(po.uniform((20, h - 2, h - 2), 95, 2 + i), 8)
                     for i in range(n)])
    got = run_conv_tf32(x, k, relu=True, skip=skip, x3=True)
    for i in range(n):
        want = np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8) + skip[i], 0)
        assert_tol(got[i], want, f"tf32x3 relu+skip img {i}")
        assert not got[i][-1][..., 4:].any(), "padded output channels must be exact 0"


@pytest.mark.parametrize("ci,co,h,w,n", [(16, 64, 34, 26, 2), (24, 264, 18, 18, 1)])
def test_tf32x3_fused_maxpool_epilogue(ci, co, h, w, n):
    """split-TF32 conv + ReLU + 2x2 max-pool in one kernel == the same conv
    followed by the bit-exact pool kernel, bit for bit."""
    l = nets.Layer("p", ci, co, h, w, 3, 3, 1)
    x = po.uniform((n, ci, h, w), 9750 + ci, co)
    k = po.uniform((ci, co, 3, 3), 9751 + ci, co)
    a = nets.Act(n, ci, h, w)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    wp = nets.prepare_tf32(l, nets.pack_weights(dev(k), False), x3=True)
    y = nets.Act(n, co, l.h_o, l.w_o)
    nets.conv_tf32(l, n, a, wp, y, _abi.EPI_RELU, x3=True)
    ref = nets.Act(n, co, l.h_o // 2, l.w_o // 2, halo=1)
    nets.maxpool_into(y, ref)
    z = nets.Act(n, co, l.h_o // 2, l.w_o // 2, halo=1)
    nets.conv_tf32(l, n, a, wp, z, _abi.EPI_RELU | _abi.EPI_MAXPOOL, x3=True)
    assert torch.equal(z.buf, ref.buf)
    for i in range(n):
        assert_tol(host(y.buf)[i], np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8), 0),
                   f"tf32x3 img {i}")


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("ci,co,h,w,n", [(16, 64, 34, 34, 2), (24, 136, 18, 66, 1), (8, 40, 10, 130, 3)])
def test_ffma_fused_maxpool_epilogue(ci, co, h, w, n, variant):
    """FFMA conv + ReLU + 2x2/s2 max-pool in one kernel (in-thread vertical
    and lane^1 horizontal window partners) equals the FFMA conv with the
    same tile followed by the bit-exact pool kernel, bit for bit; windows
    span stacked images."""
    l = nets.Layer("p", ci, co, h, w, 3, 3, 1)
    x = po.uniform((n, ci, h, w), 9800 + ci, co)
    k = po.uniform((ci, co, 3, 3), 9801 + ci, co)
    a = nets.Act(n, ci, h, w)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    wb = nets.pack_weights(dev(k), False)
    z = nets.Act(n, co, l.h_o // 2, l.w_o // 2, halo=1)
    nets.conv(l, n, a, wb, z, _abi.EPI_RELU | _abi.EPI_MAXPOOL, tile_variant=variant + 1)
    got = host(z.buf)
    for i in range(n):
        y = np.maximum(po.conv_oracle64(x[i], k, 1), 0)
        want = po.pack_feature_map(y.reshape(co, l.h_o // 2, 2, l.w_o // 2, 2).max(axis=(2, 4)), 8)
        assert_tol(got[i, :, 1:-1, 1:-1], want, f"fused pool img {i}")
        assert not got[i, :, 0].any() and not got[i, :, :, 0].any()


@pytest.mark.parametrize("ci,co,h,w,n", [(16, 64, 34, 26, 2), (24, 264, 18, 18, 1), (8, 40, 66, 10, 3)])
def test_tf32_fused_maxpool_epilogue(ci, co, h, w, n):
    """conv + ReLU + 2x2/s2 max-pool in the TF32 epilogue (the VGG pooled
    layers on the TF32 path) equals the TF32 conv followed by the separate
    bit-exact pool kernel, bit for bit, written into a halo'd view."""
    l = nets.Layer("p", ci, co, h, w, 3, 3, 1)
    x = po.uniform((n, ci, h, w), 9700 + ci, co)
    k = po.uniform((ci, co, 3, 3), 9701 + ci, co)
    a = nets.Act(n, ci, h, w)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    wp = nets.prepare_tf32(l, nets.pack_weights(dev(k), False))
    y = nets.Act(n, co, l.h_o, l.w_o)
    nets.conv_tf32(l, n, a, wp, y, _abi.EPI_RELU)
    ref = nets.Act(n, co, l.h_o // 2, l.w_o // 2, halo=1)
    nets.maxpool_into(y, ref)
    z = nets.Act(n, co, l.h_o // 2, l.w_o // 2, halo=1)
    nets.conv_tf32(l, n, a, wp, z, _abi.EPI_RELU | _abi.EPI_MAXPOOL)
    assert torch.equal(z.buf, ref.buf)
    # odd outputs: refused, not silently wrong
    lo = nets.Layer("o", ci, co, h + 1, w, 3, 3, 1)
    ao = nets.Act(n, ci, h + 1, w)
    with pytest.raises(ValueError, match="even"):
        nets.conv_tf32(lo, n, ao, nets.prepare_tf32(lo, nets.pack_weights(dev(k), False)), z,
                       _abi.EPI_MAXPOOL)


@pytest.mark.parametrize("ci,co,hb,s", [(32, 64, 56, 2), (40, 136, 27, 2), (16, 24, 13, 3)])
def test_tf32_strided_1x1_on_crop_view(ci, co, hb, s):
    """1x1 stride-s convs (ResNet projections) on the TF32 path: a stride-1
    1x1 over the tensor map's subsampled view, here of a crop view (h_i =
    hb - 1 rows/cols of an hb x hb buffer, like the 55x55 crop of 56x56)."""
    n = 2
    hi = hb - 1 if (hb - 2) % s == 0 else hb
    x = po.uniform((n, ci, hb, hb), 9900 + ci, s)
    k = po.uniform((ci, co, 1, 1), 9901 + ci, s)
    a = nets.Act(n, ci, hb, hb)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    l = nets.Layer("pr", ci, co, hi, hi, 1, 1, s)
    y = nets.Act(n, co, l.h_o, l.w_o)
    wp = nets.prepare_tf32(l, nets.pack_weights(dev(k), False))
    nets.conv_tf32(l, n, a, wp, y, in_view=a.full_view())
    got = host(y.buf)
    for i in range(n):
        xc = np.ascontiguousarray(x[i][:, :hi, :hi])
        want = po.pack_feature_map(po.conv_oracle64(xc, k, s), 8)
        err = np.abs(got[i].astype(np.float64) - want)
        bound = 2.0 ** -9 * po.pack_feature_map(po.conv_oracle64(np.abs(xc), np.abs(k), s), 8) + 1e-5
        assert (err <= bound).all(), f"max err {err.max()}"
        assert err.max() > 0  # really the TF32 path


@pytest.mark.parametrize("n,h", [(1, 12), (3, 9)])
def test_tf32_epilogue_and_padding(n, h):
    """ReLU + skip epilogue and zero padded channels; h = 9 (7x7 output)
    stacks two images per M-tile (the last unit half empty)."""
    x = po.uniform((n, 16, h, h), 93, 0)
    k = po.uniform((16, 20, 3, 3), 93, 1)
    skip = np.stack([po.pack_feature_map(po.uniform((20, h - 2, h - 2), 93, 2 + i), 8)
                     for i in range(n)])
    got = run_conv_tf32(x, k, relu=True, skip=skip)
    for i in range(n):
        want = np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8) + skip[i], 0)
        assert (np.abs(got[i] - want) <= tf32_bound(x[i], k)).all()
        assert not got[i][-1][..., 4:].any(), "padded output channels must be exact 0"


def test_tail_split_launch():
    """Unit counts just above a wave (196 units on 148 SMs): the full wave runs
    unsplit, the ragged tail as a second, split-K launch (the first unit
    ranges of each launch and the seam between them are checked)."""
    n, ci, co, hi = 16, 64, 64, 58
    x = po.uniform((n, ci, hi, hi), 9300, 0)
    k = po.uniform((ci, co, 3, 3), 9300, 1)
    l = nets.Layer("tail", ci, co, hi, hi, 3, 3, 1)
    a = nets.Act(n, ci, hi, hi)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    y = nets.Act(n, co, l.h_o, l.w_o)
    nets.conv(l, n, a, nets.pack_weights(dev(k), False), y)
    got = host(y.buf)
    kb = po.pack_kernel(k, 8, 8)
    for i in (0, 11, 12, 15):  # main-wave images and tail images
        xb = po.pack_feature_map(x[i], 8)
        for r in (0, 27, 55):
            want = po.conv_oracle64_blocked(xb, kb, ci, co, 1, r, r + 1)
            assert_tol(got[i, :, r], want[:, r], f"img {i} row {r}")


@pytest.mark.parametrize("ci,co,hi,f,n,epi", [
    (64, 128, 58, 3, 16, 0),                               # 392 units: 2.65 waves, plain
    (128, 192, 30, 3, 24, _abi.EPI_RELU),                  # ragged C_o group, ReLU
    (256, 256, 16, 1, 96, _abi.EPI_ADD | _abi.EPI_RELU),   # dense 1x1 + skip-add (epilogue warpgroup)
    (512, 512, 16, 3, 32, _abi.EPI_ADD),                   # 14x14 maps across images, 1.35 waves
    (512, 512, 30, 3, 4, _abi.EPI_ADD | _abi.EPI_RELU),    # 104 units < 148 SMs: 3-piece chains
    (512, 512, 16, 3, 8, 0),                               # 56 units: 4-piece chains (middle pieces)
])
def test_stream_k_launch(ci, co, hi, f, n, epi):
    """Ragged unit counts (1.x / 2.65 waves of 148 SMs, or fewer units than
    SMs) run as one stream-K launch: whole waves round-robin, then the last
    1.x waves (or everything) cut at stage granularity, the cut units
    finished through the output map -- through chains of middle pieces when a
    unit spans three or more CTAs.  Every
    element against the fp64 GPU referee at the fp32 tolerance; a second
    launch (flags self-reset) and a launch on another stream (its own flag
    slot) are bitwise equal to the first."""
    from oracle import gpu_oracle as go
    l = nets.Layer("sk", ci, co, hi, hi, f, f, 1)
    wd = torch.empty((ci, co, f, f), device="cuda").uniform_(-1, 1)
    a = nets.Act(n, ci, hi, hi)
    a.buf.uniform_(-1, 1)
    sk = None
    if epi & _abi.EPI_ADD:
        sk = nets.Act(n, co, l.h_o, l.w_o)
        sk.buf.uniform_(-1, 1)
    w = nets.pack_weights(wd, False)
    y = nets.Act(n, co, l.h_o, l.w_o)
    launches = _abi.lib().dconv_cuda_launch_count()
    nets.conv(l, n, a, w, y, epi, sk)
    torch.cuda.synchronize()
    # one launch: not the full waves + split-K tail pair
    assert _abi.lib().dconv_cuda_launch_count() - launches == 1
    want = go.conv64_act(a, l, wd)
    if sk is not None:
        want = want + sk.buf.double()
    if epi & _abi.EPI_RELU:
        want = want.clamp_min(0.0)
    ok, nbad, err, ratio = go.check_tol(y.buf, want)
    assert ok, f"{nbad} elements out of tolerance, max err {err}"
    first = y.buf.clone()
    y.buf.fill_(float("nan"))
    nets.conv(l, n, a, w, y, epi, sk)
    torch.cuda.synchronize()
    assert torch.equal(y.buf, first), "second launch differs (flag not reset?)"
    side = torch.cuda.Stream()
    y.buf.fill_(float("nan"))
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        nets.conv(l, n, a, w, y, epi, sk, stream=side)
    side.synchronize()
    assert torch.equal(y.buf, first), "launch on a second stream differs"


@pytest.mark.parametrize("cb", [16, 32])
@pytest.mark.parametrize("ci,co,hi,f,n", [(64, 128, 58, 3, 16), (256, 256, 16, 1, 96)])
def test_stream_k_wide_channel_blocks(cb, ci, co, hi, f, n):
    """Stream-K launches (ragged unit counts) with c_ib = c_ob = 16 / 32
    storage blocks -- the 3x3 loop and the dense 1x1 loop, skip-add + ReLU --
    every element against the fp64 GPU referee."""
    from oracle import gpu_oracle as go
    xd = torch.empty((n, ci, hi, hi), device="cuda").uniform_(-1, 1)
    wd = torch.empty((ci, co, f, f), device="cuda").uniform_(-1, 1)
    shape = D.ConvShape(ci, co, hi, hi, f, f, 1)
    xb = D.pack_feature_map(xd, cb)
    kb = D.pack_kernel(wd, cb, cb)
    skd = torch.empty((n, co, shape.h_o, shape.w_o), device="cuda").uniform_(-1, 1)
    sk = D.pack_feature_map(skd, cb)
    launches = _abi.lib().dconv_cuda_launch_count()
    y = D.conv_direct(xb, kb, shape, D.BlockingParams(cb, 1, cb), relu=True, skip=sk,
                      algo=_abi.ALGO_FFMA)
    torch.cuda.synchronize()
    assert _abi.lib().dconv_cuda_launch_count() - launches == 1
    want = go.conv64(xd.data_ptr(), n, ci, hi, hi, 1, ci * hi * hi, hi * hi, hi, wd, 1)
    want = (want + D.pack_feature_map(skd, 8).data.double()).clamp_min(0.0)
    # c_b-blocked output -> blocks of 8 channels
    got = y.data.view(n, co // cb, shape.h_o, shape.w_o, cb // 8, 8).permute(0, 1, 4, 2, 3, 5)
    got = got.reshape(n, co // 8, shape.h_o, shape.w_o, 8)
    ok, nbad, err, ratio = go.check_tol(got, want)
    assert ok, f"c_b {cb}: {nbad} elements out of tolerance, max err {err}"


def test_first_launch_under_graph_capture():
    """A fresh process whose very first conv launch (a stream-K one) happens
    under CUDA-graph capture: the launcher's one-time set-up (kernel
    attributes, cluster occupancy, the stream-K flag lookup) is legal there,
    and two replays give the eager result bitwise."""
    import os
    import subprocess
    import sys
    code = r"""
import torch, sys
sys.path.insert(0, ".")
from paper_1809_10170_b200 import nets
n, ci, co, hi = 16, 64, 128, 58
l = nets.Layer("cap", ci, co, hi, hi, 3, 3, 1)
a = nets.Act(n, ci, hi, hi); a.buf.uniform_(-1, 1)
w = nets.pack_weights(torch.empty((ci, co, 3, 3), device="cuda").uniform_(-1, 1), False)
y = nets.Act(n, co, l.h_o, l.w_o)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    nets.conv(l, n, a, w, y, stream=torch.cuda.current_stream())
g.replay(); g.replay(); torch.cuda.synchronize()
got = y.buf.clone(); y.buf.zero_()
nets.conv(l, n, a, w, y); torch.cuda.synchronize()
assert torch.equal(got, y.buf) and float(got.abs().max()) > 0
print("capture ok")
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "capture ok" in r.stdout, r.stdout + r.stderr


def test_output_pencil_alignment_contract():
    """The fast kernels move output / skip pencils by 256-bit accesses: an
    output view at a 16-byte but not 32-byte aligned address runs on the
    generic kernel under ALGO_AUTO (same result within the tolerance) and is
    refused with DCONV_EUNSUPPORTED when the FFMA kernel is forced."""
    import ctypes
    ci, co, hi = 16, 24, 12
    x = po.uniform((ci, hi, hi), 9500, 0)
    k = po.uniform((ci, co, 3, 3), 9500, 1)
    shape = D.ConvShape(ci, co, hi, hi, 3, 3, 1)
    xb = D.BlockedFeatureMap(ci, hi, hi, 8, data=dev(po.pack_feature_map(x, 8)[None]))
    kb = D.BlockedKernel(ci, co, 3, 3, 8, 8, data=dev(po.pack_kernel(k, 8, 8)))
    n_out = 3 * shape.h_o * shape.w_o * 8
    buf = torch.zeros(n_out + 8, dtype=torch.float32, device="cuda")
    assert buf.data_ptr() % 32 == 0
    out = buf[4:4 + n_out]  # 16-byte aligned, not pencil-aligned
    want = po.pack_feature_map(po.conv_oracle64(x, k, 1), 8)
    for algo, ok in ((_abi.ALGO_AUTO, True), (_abi.ALGO_FFMA, False)):
        d = D.make_desc(shape, 1, 8, 8, 0, algo)
        rc = _abi.lib().dconv_cuda_conv_direct(ctypes.byref(d), _abi.ptr(xb.data), _abi.ptr(kb.data),
                                               0, out.data_ptr(), _abi.stream_ptr(None))
        if ok:
            assert rc == _abi.OK, _abi.lib().dconv_cuda_last_error_detail()
            assert_tol(host(out).reshape(want.shape), want, "generic kernel on the unaligned view")
        else:
            assert rc == _abi.EUNSUPPORTED
            assert b"pencil-aligned" in _abi.lib().dconv_cuda_last_error_detail()


def test_autotuned_plan_matches_default_tiles():
    """Per-layer tile autotune changes only the CTA tiling: every layer output
    stays within tolerance of the default-tile run (tile choices differ in
    fp32 summation order, not in math)."""
    a = nets.build_plan("googlenet", 2, seed=11)
    b = nets.build_plan("googlenet", 2, seed=11)
    tiles = b.autotune()
    assert set(tiles.values()) <= {1, 2, 3, 4}
    a.run()
    b.run()
    torch.cuda.synchronize()
    for name in a.outputs:
        x, y = host(a.outputs[name].buf), host(b.outputs[name].buf)
        scale = max(1.0, float(np.abs(x).max()))
        assert float(np.abs(x - y).max()) <= 1e-5 * scale + 1e-4, name


def test_tf32_plans_read_the_stride1_first_layer_in_place():
    """Tensor-core plans run VGG's stride-1 first layer on the FFMA
    first-layer reader (dense image read in place: no padded copy, no pack
    launch); its output is the FFMA plan's, bit for bit."""
    a = nets.build_plan("vgg16", 1, seed=13)
    for algo in ("tf32", "tf32x3"):
        b = nets.build_plan("vgg16", 1, seed=13, algo=algo)
        assert b.steps[0].kind == "first" and not any(s.kind == "pack" for s in b.steps)
        a.run()
        b.run()
        torch.cuda.synchronize()
        assert torch.equal(a.outputs["conv1_1"].buf, b.outputs["conv1_1"].buf), algo


@pytest.mark.parametrize("config,name", [("googlenet", "conv1_7x7_s2"), ("alexnet", "conv1")])
def test_tf32_space_to_depth_stem_matches_reader(config, name):
    """TF32 plans run strided stems as space-to-depth repack + stride-1
    tcgen05 conv; the result equals the fp32 first-layer reader within the
    TF32 bound (the s2d weights are an exact rearrangement, extra taps zero)."""
    a = nets.build_plan(config, 1, seed=17)
    b = nets.build_plan(config, 1, seed=17, algo="tf32")
    assert any(s.kind == "pack" and s.name == f"pack_{name}" for s in b.steps)
    a.run()
    b.run()
    torch.cuda.synchronize()
    l = [x for x in a.layers if x.name == name][0]
    ya, yb = host(a.outputs[name].buf), host(b.outputs[name].buf)
    x = host(a.input)[0]
    k = po.unpack_kernel(host(a.weights[name]), l.c_i, l.c_o)
    bound = 2.0 ** -9 * po.pack_feature_map(po.conv_oracle64(np.abs(x), np.abs(k), l.s), 8) + 1e-5
    assert (np.abs(ya[0] - yb[0]) <= 2 * bound).all()
    assert np.abs(ya[0] - yb[0]).max() > 0  # the tcgen05 path really ran


@pytest.mark.parametrize("algo", ["tf32", "tf32x3"])
def test_tensor_core_strided_layers_read_space_to_depth_in_place(algo, monkeypatch):
    """ResNet-50's 3x3/s2 convs on the tensor-core paths: computed as stride-1
    layers over the space-to-depth view of the (top/left-padded) input, read
    in place by strided TMA -- the plan has no repack step -- and equal to
    the fp64 oracle within the TF32 bound (tf32) or the chain's normwise fp32
    bound (tf32x3; deep unnormalised activations, as the full-size chain
    checks) on every row of the output (teacher-forced: the plan's own
    input).  Batch 2 with the batch-1 FFMA routing of split-TF32 plans off."""
    monkeypatch.setattr(nets.Plan, "_few_units", lambda self, l, epi: False)
    b = nets.build_plan("resnet50", 2, seed=19, algo=algo)
    assert not any(st.name.startswith("s2d_") for st in b.steps)
    rec = {}
    orig = nets.conv_tf32

    def spy(l, n, x, wp, out, epilogue=0, skip=None, stream=None, in_view=None, **kw):
        orig(l, n, x, wp, out, epilogue, skip, stream, in_view, **kw)
        torch.cuda.synchronize()
        if l.s > 1 and l.h_f > 1:
            rec[l.name] = (l, host(x.buf), host(out.buf), out, epilogue)
            calls[l.name] = (l, n, x, wp, out, epilogue, skip, in_view, kw)
    calls = {}
    nets.conv_tf32 = spy
    try:
        b.run()
    finally:
        nets.conv_tf32 = orig
    assert sorted(rec) == ["s2b1_c2", "s3b1_c2", "s4b1_c2"]
    if algo == "tf32x3":
        # per element at the fp32 tolerance: the same launches (in-place
        # strided TMA) on fresh uniform[-1,1] inputs, where the bound applies
        for name, (l, n, x, wp, out, epilogue, skip, in_view, kw) in calls.items():
            nets._fill(x.buf, 77, len(name))
            orig(l, n, x, wp, out, epilogue, skip, None, in_view, **kw)
            xs, ys = host(x.buf), host(out.buf)
            kb = po.pack_kernel(po.unpack_kernel(host(b.weights[name]), l.c_i, l.c_o), 8, 8)
            for i in range(2):
                xb = np.ascontiguousarray(xs[i][:, :l.h_i, :l.w_i, :])
                want = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, 0, l.h_o)
                if epilogue & _abi.EPI_RELU:
                    want = np.maximum(want, 0)
                got = ys[i][:, out.halo:out.halo + l.h_o, out.halo:out.halo + l.w_o]
                assert_tol(got, want, f"{name} fresh input img {i}")
    for name, (l, xs, ys, out, epi) in rec.items():
        kb = po.pack_kernel(po.unpack_kernel(host(b.weights[name]), l.c_i, l.c_o), 8, 8)
        for i in range(2):
            xb = np.ascontiguousarray(xs[i][:, :l.h_i, :l.w_i, :])
            want = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, 0, l.h_o)
            if epi & _abi.EPI_RELU:
                want = np.maximum(want, 0)
            got = ys[i][:, out.halo:out.halo + l.h_o, out.halo:out.halo + l.w_o]
            if algo == "tf32x3":
                scale = max(1.0, float(np.abs(want).max()))
                err = float(np.abs(got - want).max())
                assert err <= 1e-5 * scale + 1e-4, f"{name} img {i}: err {err} scale {scale}"
            else:
                bound = 2.0 ** -9 * po.conv_oracle64_blocked(np.abs(xb), np.abs(kb), l.c_i, l.c_o,
                                                             l.s, 0, l.h_o) + 1e-5
                assert (np.abs(got - want) <= bound).all(), name


@pytest.mark.parametrize("x3", [False, True])
@pytest.mark.parametrize("ci,co,h,f,s,n", [(64, 72, 21, 3, 2, 2), (24, 256, 17, 5, 2, 1),
                                            (16, 64, 27, 3, 3, 2), (40, 136, 15, 3, 2, 3),
                                            (8, 96, 59, 11, 4, 2), (64, 128, 57, 5, 4, 8)])
def test_tensor_core_strided_kxk_through_the_abi(ci, co, h, f, s, n, x3):
    """k x k stride-s layers straight through the tensor-core C-ABI (in-place
    space-to-depth, ragged channel counts, stride 3, stacked 7x7 tiles)."""
    l = nets.Layer("s", ci, co, h, h, f, f, s)
    x = po.uniform((n, ci, h, h), 9950 + ci, s)
    k = po.uniform((ci, co, f, f), 9951 + ci, s)
    a = nets.Act(n, ci, h, h)
    a.buf.copy_(dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
    wp = nets.prepare_tf32(l, nets.pack_weights(dev(k), False), x3=x3)
    y = nets.Act(n, co, l.h_o, l.w_o)
    nets.conv_tf32(l, n, a, wp, y, _abi.EPI_RELU, x3=x3)
    got = host(y.buf)
    for i in range(n):
        want = np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, s), 8), 0)
        if x3:
            assert_tol(got[i], want, f"img {i}")
        else:
            bound = 2.0 ** -9 * po.pack_feature_map(po.conv_oracle64(np.abs(x[i]), np.abs(k), s), 8)
            assert (np.abs(got[i] - want) <= bound + 1e-5).all()
        assert np.abs(got[i] - want).max() > 0  # the tensor-core path really ran


def test_tensor_core_rejects_stride_over_8():
    """Strides > 8 exceed the TMA element-stride limit: a clear
    EUNSUPPORTED, not a tensor-map encode failure."""
    l = nets.Layer("s9", 8, 8, 28, 28, 10, 10, 9)
    a = nets.Act(1, 8, 28, 28)
    y = nets.Act(1, 8, l.h_o, l.w_o)
    for x3 in (False, True):
        with pytest.raises(RuntimeError, match="stride"):
            wp = nets.prepare_tf32(l, nets.pack_weights(dev(po.uniform((8, 8, 10, 10), 1, 2)),
                                                        False), x3=x3)
            nets.conv_tf32(l, 1, a, wp, y, x3=x3)


@pytest.mark.parametrize("config,n", [("vgg16", 32), ("resnet50", 256), ("googlenet", 64)])
def test_full_size_plans_sampled_parity(config, n):
    """The bench workloads at their full BASELINE batch (every tile shape,
    tail split and epilogue-warpgroup path the bench runs): each conv layer's
    output for the first, a middle and the last image, on three rows, against
    the fp64 oracle on the same (teacher-forced) inputs.  Independent-layer
    configs (uniform[-1,1] inputs) use the per-element fp32 bound; the deep
    unnormalised chains use the normwise form of it per layer (activations
    grow with depth, so near-zero outputs of large cancelling sums carry
    fp32 rounding of the large terms -- SURVEY §7.4.4, as the chain test)."""
    normwise = config in ("vgg16", "resnet50")

    def check(g, want, what):
        if not normwise:
            assert_tol(g, want, what)
            return
        scale = max(1.0, float(np.abs(want).max()))
        err = float(np.abs(g - want).max())
        assert err <= 1e-5 * scale + 1e-4, f"{what}: err {err} scale {scale}"
    plan = nets.build_plan(config, n, seed=23)
    imgs = sorted({0, n // 2, n - 1})
    rec = []
    orig = nets.conv

    def spy(l, nn, x, w, out, epilogue=0, skip=None, stream=None, in_view=None, co_range=None,
            **kw):
        orig(l, nn, x, w, out, epilogue, skip, stream, in_view, co_range, **kw)
        torch.cuda.synchronize()
        xt = x if isinstance(x, torch.Tensor) else x.buf
        rec.append((l, xt[imgs].cpu(), out.buf[imgs].cpu(), out, epilogue,
                    skip.buf[imgs].cpu() if skip is not None else None, skip, w))
    nets.conv = spy
    try:
        plan.run()
    finally:
        nets.conv = orig
    assert len(rec) == len(plan.layers)
    _check_sampled(config, [(l, xin, yout, out, epi, skb, skip,
                             po.pack_kernel(po.unpack_kernel(host(w), l.c_i, l.c_o), 8, 8))
                            for l, xin, yout, out, epi, skb, skip, w in rec], imgs, check)


def _check_sampled(config, rec, imgs, check):
    """Sampled rows of every recorded launch (input, output, epilogue of the
    first / middle / last image) against the fp64 oracle on the same input."""
    for l, xin, yout, out, epi, skb, skip, kb in rec:
        for j in range(len(imgs)):
            x = xin[j].numpy()
            xb = (po.pack_feature_map(np.ascontiguousarray(x[:, :l.h_i, :l.w_i]), 8) if l.first
                  else np.ascontiguousarray(x[:, :l.h_i, :l.w_i, :]))
            got = yout[j].numpy()
            h = out.halo
            if epi & _abi.EPI_MAXPOOL:
                hp, wp = l.h_o // 2, l.w_o // 2
                for rp in sorted({0, hp // 2, hp - 1}):
                    two = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, 2 * rp, 2 * rp + 2)
                    two = np.maximum(two[:, 2 * rp:2 * rp + 2], 0)
                    want = two.reshape(two.shape[0], 2, wp, 2, 8).max(axis=(1, 3))
                    check(got[:, h + rp, h:h + wp, :], want, f"{config}/{l.name} img {imgs[j]}")
                continue
            for r in sorted({0, l.h_o // 2, l.h_o - 1}):
                want = po.conv_oracle64_blocked(xb, kb, l.c_i, l.c_o, l.s, r, r + 1)[:, r]
                if epi & _abi.EPI_ADD:
                    sk = skb[j].numpy()
                    want = want + sk[:, skip.halo + r, skip.halo:skip.halo + l.w_o, :]
                if epi & _abi.EPI_RELU:
                    want = np.maximum(want, 0)
                check(got[:, h + r, h:h + l.w_o, :], want, f"{config}/{l.name} img {imgs[j]} row {r}")


@pytest.mark.parametrize("config,n", [("vgg16", 32), ("resnet50", 256), ("googlenet", 64)])
def test_tf32x3_full_size_plans_sampled_parity(config, n):
    """The split-TF32 bench workloads at full batch: every tensor-core launch
    (space-to-depth stems and strided layers, fused pools, skip-add
    epilogues, image-stacked 7x7 tiles) checked on sampled rows of the
    first / middle / last image against the fp64 oracle with the same fp32
    bound as the FFMA plans (per element for independent layers, per layer
    normwise for the deep chains)."""
    normwise = config in ("vgg16", "resnet50")

    def check(g, want, what):
        if not normwise:
            assert_tol(g, want, what)
            return
        scale = max(1.0, float(np.abs(want).max()))
        err = float(np.abs(g - want).max())
        assert err <= 1e-5 * scale + 1e-4, f"{what}: err {err} scale {scale}"
    prepared = {}
    orig_prep, orig_conv = nets.prepare_tf32, nets.conv_tf32

    def prep_spy(l, w_blocked, stream=None, x3=False):
        wp = orig_prep(l, w_blocked, stream, x3)
        prepared[wp.data_ptr()] = host(w_blocked).copy()
        return wp
    nets.prepare_tf32 = prep_spy
    try:
        plan = nets.build_plan(config, n, seed=29, algo="tf32x3")
    finally:
        nets.prepare_tf32 = orig_prep
    imgs = sorted({0, n // 2, n - 1})
    rec = []

    def spy(l, nn, x, wp, out, epilogue=0, skip=None, stream=None, in_view=None, x3=False):
        assert x3
        orig_conv(l, nn, x, wp, out, epilogue, skip, stream, in_view, x3=x3)
        torch.cuda.synchronize()
        kb = po.pack_kernel(po.unpack_kernel(prepared[wp.data_ptr()], l.c_i, l.c_o), 8, 8)
        rec.append((l, x.buf[imgs].cpu(), out.buf[imgs].cpu(), out, epilogue,
                    skip.buf[imgs].cpu() if skip is not None else None, skip, kb))
    nets.conv_tf32 = spy
    try:
        plan.run()
    finally:
        nets.conv_tf32 = orig_conv
    assert len(rec) == sum(1 for st in plan.steps if st.kind == "tf32") > 0
    _check_sampled(config, rec, imgs, check)


def test_python_dropin_tensor_core_conv():
    """dconv.PreparedKernel + conv_direct_tc (the Python mirror of the C++
    DevicePreparedKernel overload): split-TF32 meets conv_direct's fp32
    tolerance with ReLU + skip; the single-pass TF32 kernel meets its own."""
    ci, co, h = 256, 72, 11
    x = po.uniform((2, ci, h, h), 9601, 0)
    k = po.uniform((ci, co, 3, 3), 9602, 0)
    skip = np.stack([po.pack_feature_map(po.uniform((co, h - 2, h - 2), 9603, i), 8)
                     for i in range(2)])
    shape = D.ConvShape(ci, co, h, h, 3, 3, 1)
    xb = D.BlockedFeatureMap(ci, h, h, 8, n=2,
                             data=dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(2)])))
    kb = D.BlockedKernel(ci, co, 3, 3, 8, 8, data=dev(po.pack_kernel(k, 8, 8)))
    sk = D.BlockedFeatureMap(co, h - 2, h - 2, 8, n=2, data=dev(skip))
    y3 = host(D.conv_direct_tc(xb, D.PreparedKernel(kb, shape, split=True), relu=True, skip=sk).data)
    y1 = host(D.conv_direct_tc(xb, D.PreparedKernel(kb, shape, split=False)).data)
    for i in range(2):
        ref = po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8)
        assert_tol(y3[i], np.maximum(ref + skip[i], 0), f"split-TF32 img {i}")
        assert (np.abs(y1[i] - ref) <= tf32_bound(x[i], k)).all()
    with pytest.raises(ValueError, match="layout error"):
        D.PreparedKernel(D.BlockedKernel(ci, co, 3, 3, 8, 4), shape)


def test_space_to_depth_blocked_bitexact():
    """dconv_cuda_space_to_depth_blocked (C-ABI utility; the tensor-core
    kernels read this view in place instead): channel (dy*f + dx)*C + c at
    (y, x) is pixel (f*y + dy, f*x + dx), zero outside, bit-exact."""
    n, c, h, w, f = 2, 16, 9, 11, 2
    x = po.uniform((n, c, h, w), 9960, 0)
    xb = dev(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)]))
    hs, ws = -(-h // f), -(-w // f)
    out = torch.empty((n, (c * f * f + 7) // 8, hs, ws, 8), device="cuda")
    blk = h * w * 8
    _abi.check(_abi.lib().dconv_cuda_space_to_depth_blocked(
        _abi.ptr(xb), 2 * blk, blk, w * 8, n, c, h, w, f, _abi.ptr(out), _abi.stream_ptr()))
    got = host(out)
    for i in range(n):
        xp = np.zeros((c, hs * f, ws * f), np.float32)
        xp[:, :h, :w] = x[i]
        want = np.zeros((c * f * f, hs, ws), np.float32)
        for dy in range(f):
            for dx in range(f):
                want[(dy * f + dx) * c:(dy * f + dx + 1) * c] = xp[:, dy::f, dx::f]
        assert np.array_equal(got[i], po.pack_feature_map(want, 8))


@pytest.mark.parametrize("c,f,h,w", [(3, 2, 229, 229), (3, 2, 9, 12), (3, 4, 227, 227),
                                     (3, 3, 13, 10), (5, 2, 9, 11)])
def test_pack_space_to_depth_bitexact(c, f, h, w):
    """dconv_cuda_pack_space_to_depth (the tensor-core plans' strided-stem
    pack of the dense image): s2d channel (dy*f + dx)*C + c at (ys, xs) is
    input (c, f*ys + dy, f*xs + dx), zero outside the image and in the pad
    channels, blocked by 8 -- bit-exact (C = 3, f = 2 / 4: the per-pixel
    kernel; other shapes: the per-element one)."""
    n = 3
    x = po.uniform((n, c, h, w), 9970 + f, 0)
    hs, ws = -(-h // f), -(-w // f)
    out = torch.full((n, (c * f * f + 7) // 8, hs, ws, 8), float("nan"), device="cuda")
    _abi.check(_abi.lib().dconv_cuda_pack_space_to_depth(
        _abi.ptr(dev(x)), n, c, h, w, f, _abi.ptr(out), _abi.stream_ptr()))
    got = host(out)
    for i in range(n):
        xp = np.zeros((c, hs * f, ws * f), np.float32)
        xp[:, :h, :w] = x[i]
        want = np.zeros((c * f * f, hs, ws), np.float32)
        for dy in range(f):
            for dx in range(f):
                want[(dy * f + dx) * c:(dy * f + dx + 1) * c] = xp[:, dy::f, dx::f]
        assert np.array_equal(got[i], po.pack_feature_map(want, 8))


@pytest.mark.parametrize("f,s,h,w,co,n", [(3, 1, 34, 45, 64, 40), (3, 1, 20, 226, 40, 30),
                                           (7, 2, 41, 39, 96, 36), (7, 2, 229, 229, 64, 6),
                                           (3, 1, 226, 226, 72, 3)])
def test_first_layer_tma_reader_every_element(f, s, h, w, co, n):
    """The TMA-store first-layer reader (conv_reader.cu; many-tile layers):
    ragged tiles in both directions (clipped by the tensor store), partial
    and multiple 64-channel groups, a halo'd output view, ReLU -- every
    element against the fp64 GPU referee, and bitwise equal to the
    register-tiled reader it replaces except for summation order (both
    within the fp32 bound)."""
    from oracle import gpu_oracle as go
    l = nets.Layer("r", 3, co, h, w, f, f, s, first=True)
    xd = torch.empty((n, 3, h, w), device="cuda")
    nets._fill(xd, 61 + f, co)
    wd = torch.empty((3, co, f, f), device="cuda")
    nets._fill(wd, 62 + f, co)
    wb = nets.pack_weights(wd, True)
    y = nets.Act(n, co, l.h_o, l.w_o, halo=1)
    before = _abi.lib().dconv_cuda_launch_count()
    nets.conv(l, n, xd, wb, y, _abi.EPI_RELU)
    torch.cuda.synchronize()
    want = go.conv64_act(xd, l, wd).clamp_min(0.0)
    ok, nbad, err, ratio = go.check_tol(y.buf[:, :, 1:-1, 1:-1, :], want)
    assert ok, f"{nbad} bad, max err {err}"
    # halo ring untouched
    assert not y.buf[:, :, 0].any() and not y.buf[:, :, -1].any()
    assert not y.buf[:, :, :, 0].any() and not y.buf[:, :, :, -1].any()
    assert _abi.lib().dconv_cuda_launch_count() == before + 1


@pytest.mark.parametrize("cb", [16, 32])
@pytest.mark.parametrize("tv", [0, 1, 2])
def test_ffma_wide_channel_blocks(cb, tv, monkeypatch):
    """c_ib = c_ob = 16 / 32 (the reference's wider BlockingParams,
    micro_kernel.hpp:43-46) on the FFMA kernel: 64- / 128-byte pencils staged
    whole, walked as 8-channel sub-blocks; ragged C_i / C_o (padded storage
    blocks), strides, 1x1 / 3x3 / 5x5 filters, ReLU and skip-add epilogues,
    the selector, each CTA tile and forced split-K -- against conv_oracle64."""
    cases = [(64, 64, 30, 30, 3, 1, 2), (40, 72, 17, 23, 5, 1, 1), (96, 80, 13, 31, 1, 2, 3),
             (200, 48, 9, 9, 3, 2, 2), (512, 128, 16, 16, 3, 1, 1), (24, 136, 12, 12, 1, 1, 4)]
    if tv == 2:
        monkeypatch.setenv("DCONV_KSPLIT", "4")
    for t, (ci, co, hi, wi, f, s, n) in enumerate(cases):
        x = po.uniform((n, ci, hi, wi), 7700 + t, cb)
        k = po.uniform((ci, co, f, f), 7710 + t, cb)
        shape = D.ConvShape(ci, co, hi, wi, f, f, s)
        xb = D.BlockedFeatureMap(ci, hi, wi, cb, n=n, data=dev(np.stack(
            [po.pack_feature_map(x[i], cb) for i in range(n)])))
        kb = D.BlockedKernel(ci, co, f, f, cb, cb, data=dev(po.pack_kernel(k, cb, cb)))
        skip_np = np.stack([po.pack_feature_map(po.uniform((co, shape.h_o, shape.w_o), 7720 + t, i),
                                                cb) for i in range(n)])
        sk = D.BlockedFeatureMap(co, shape.h_o, shape.w_o, cb, n=n, data=dev(skip_np))
        y = D.conv_direct(xb, kb, shape, D.BlockingParams(cb, 1, cb), relu=True, skip=sk,
                          algo=_abi.ALGO_FFMA, tile_variant=tv)
        got = host(y.data)
        for i in range(n):
            want = np.maximum(po.pack_feature_map(po.conv_oracle64(x[i], k, s), cb) + skip_np[i], 0)
            assert_tol(got[i], want, f"c_b {cb} tile {tv} case {t} img {i}")


@pytest.mark.parametrize("f,s,h,co,n", [(11, 4, 227, 96, 1), (7, 2, 229, 64, 1), (3, 1, 226, 64, 1),
                                         (11, 4, 51, 40, 3), (3, 1, 30, 72, 2)])
def test_first_layer_tma_reader_few_tiles(f, s, h, co, n):
    """The TMA-store reader's few-tile form (2 accumulator rows per thread:
    batch-1 stems incl. AlexNet's 11x11/s4) -- every element against the
    fp64 GPU referee, halo untouched."""
    from oracle import gpu_oracle as go
    l = nets.Layer("r", 3, co, h, h, f, f, s, first=True)
    xd = torch.empty((n, 3, h, h), device="cuda")
    nets._fill(xd, 71 + f, co)
    wd = torch.empty((3, co, f, f), device="cuda")
    nets._fill(wd, 72 + f, co)
    y = nets.Act(n, co, l.h_o, l.w_o, halo=1)
    nets.conv(l, n, xd, nets.pack_weights(wd, True), y, _abi.EPI_RELU)
    torch.cuda.synchronize()
    want = go.conv64_act(xd, l, wd).clamp_min(0.0)
    ok, nbad, err, ratio = go.check_tol(y.buf[:, :, 1:-1, 1:-1, :], want)
    assert ok, f"{nbad} bad, max err {err}"
    assert not y.buf[:, :, 0].any() and not y.buf[:, :, :, -1].any()


@pytest.mark.parametrize("config", ["vgg16", "googlenet"])
def test_pipeline_streams_batches(config):
    """nets.Pipeline (the streaming e2e path): copies of neighbouring batches
    overlap the kernels, yet every batch's result is the plan's own.  The
    host input is then halved: conv, ReLU and max-pool are positively
    homogeneous and x/2 is exact, so the streamed result must be exactly half
    -- a stale input buffer or an early copy-out would show."""
    plan = nets.build_plan(config, 2, seed=44)
    plan.run()
    torch.cuda.synchronize()
    ref = [t.clone() for t in plan.io_outputs()]
    h_in = [t.cpu().pin_memory() for t in plan.io_inputs()]
    h_out = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in plan.io_outputs()]
    pipe = nets.Pipeline(plan, h_in, h_out)
    pipe.run(3)
    torch.cuda.synchronize()
    for h, r in zip(h_out, ref):
        assert torch.equal(h, r.cpu())
    for h in h_in:
        h.mul_(0.5)
    pipe.run(2)
    torch.cuda.synchronize()
    for h, r in zip(h_out, ref):
        assert torch.equal(h, (0.5 * r).cpu())
