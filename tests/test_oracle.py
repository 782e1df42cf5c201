"""CPU tests: pin the oracle (oracle/oracle.c) against the reference's own
code (oracle/_ref, compiled from /root/reference) and its golden fixtures,
and restate the SPEC.md known-answer examples.  No GPU needed."""
import ctypes
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    g = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in g.files})
    return g, names


# ---------------------------------------------------------------- layouts
def test_pack_feature_map_spec_examples():
    # SPEC.md:81-83
    assert po.pack_feature_map(np.array([[[5.0]]], np.float32), 1).ravel().tolist() == [5.0]
    x = np.array([[[1.0]], [[2.0]]], np.float32)
    assert po.pack_feature_map(x, 2).ravel().tolist() == [1.0, 2.0]
    x3 = po.uniform((3, 2, 2), 1, 0)
    b = po.pack_feature_map(x3, 4)
    assert b.size == 16 and np.all(b[..., 3] == 0.0)


def test_unpack_feature_map_roundtrip():
    # SPEC.md:91-93
    x = po.uniform((3, 5, 7), 2, 0)
    for cb in (1, 2, 4, 8):
        assert np.array_equal(po.unpack_feature_map(po.pack_feature_map(x, cb), 3), x)


def test_pack_kernel_offset_17():
    # c_i=4, c_o=8, 1x1, c_ob=c_ib=4, weight (i=0, j=5) -> 17
    k = np.zeros((4, 8, 1, 1), np.float32)
    k[0, 5, 0, 0] = 7.0
    kb = po.pack_kernel(k, 4, 4)
    assert np.flatnonzero(kb.ravel()).tolist() == [17]
    r = po.ref()
    if r is not None:
        assert r.ref_blocked_kernel_offset(4, 8, 1, 1, 4, 4, 1, 0, 0, 0, 0, 1) == 17


def test_pack_kernel_enumeration_order():
    # c_i=c_o=2, 1x1, c_ob=c_ib=1 -> [j'0:i'0, j'0:i'1, j'1:i'0, j'1:i'1]
    k = np.array([[[[1.0]], [[2.0]]], [[[3.0]], [[4.0]]]], np.float32)  # k[i][j]
    kb = po.pack_kernel(k, 1, 1).ravel().tolist()
    assert kb == [k[0, 0, 0, 0], k[1, 0, 0, 0], k[0, 1, 0, 0], k[1, 1, 0, 0]]


@pytest.mark.parametrize("cob,cib", [(1, 1), (4, 2), (8, 4), (3, 5), (16, 16)])
def test_pack_kernel_roundtrip(cob, cib):
    # SPEC.md:103, :109-111
    k = po.uniform((3, 5, 3, 3), 3, cob * 31 + cib)
    assert np.array_equal(po.unpack_kernel(po.pack_kernel(k, cob, cib), 3, 5), k)


def test_layout_roundtrips_random():
    # acceptance 7, scaled down
    rng = np.random.default_rng(7)
    for t in range(60):
        c, h, w = rng.integers(1, 9, 3)
        cb = int(rng.integers(1, 17))
        x = po.uniform((c, h, w), 4, t)
        assert np.array_equal(po.unpack_feature_map(po.pack_feature_map(x, cb), c), x)
        ci, co = rng.integers(1, 7, 2)
        k = po.uniform((ci, co, 2, 3), 5, t)
        cob, cib = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        assert np.array_equal(po.unpack_kernel(po.pack_kernel(k, cob, cib), ci, co), k)


# ---------------------------------------------------------------- shapes
def test_conv_shape_rules():
    assert po.conv_shape(64, 64, 58, 58, 3, 3, 1) == (56, 56)
    assert po.conv_shape(3, 96, 227, 227, 11, 11, 4) == (55, 55)
    assert po.conv_shape(3, 64, 229, 229, 7, 7, 2) == (112, 112)
    with pytest.raises(ValueError):  # BASELINE cfg5 stem at 230 (shape.cpp:36)
        po.conv_shape(3, 64, 230, 230, 7, 7, 2)
    with pytest.raises(ValueError):
        po.conv_shape(1, 1, 2, 2, 3, 3, 1)
    with pytest.raises(ValueError):
        po.conv_shape(0, 1, 2, 2, 1, 1, 1)


def test_conv_flops_spec():
    # SPEC.md:197-199
    assert po.orc().orc_conv_flops(1, 1, 1, 1, 1, 1) == 2
    assert po.orc().orc_conv_flops(3, 2, 3, 3, 2, 2) == 432


# ---------------------------------------------------------------- convolution
def test_conv_trivial_examples():
    # SPEC.md:159-161, :179
    assert po.conv_oracle64(np.array([[[2.0]]], np.float32),
                            np.array([[[[3.0]]]], np.float32), 1).item() == 6.0
    assert po.conv_oracle64(np.ones((1, 3, 3), np.float32),
                            np.ones((1, 1, 3, 3), np.float32), 1).item() == 9.0
    assert po.conv_oracle64(np.array([[[1.0]], [[2.0]]], np.float32),
                            np.array([[[[3.0]]], [[[4.0]]]], np.float32), 1).item() == 11.0
    x = po.uniform((3, 6, 6), 9, 0)
    assert not po.conv_oracle64(x, np.zeros((3, 2, 3, 3), np.float32), 1).any()


def test_golden_reproduced_by_oracle(golden):
    """oracle.c reproduces the reference's outputs bit-for-bit."""
    g, names = golden
    for n in names:
        ci, co, hi, wi, hf, wf, s, cib, cob = g[f"{n}/geom"].tolist()
        x, k = g[f"{n}/x"], g[f"{n}/k"]
        assert np.array_equal(po.conv_oracle64(x, k, s), g[f"{n}/y_oracle64"]), n
        assert np.array_equal(po.conv_naive(x, k, s), g[f"{n}/y_naive"]), n
        assert np.array_equal(po.pack_feature_map(x, cib), g[f"{n}/x_blocked"]), n
        assert np.array_equal(po.pack_kernel(k, cob, cib), g[f"{n}/k_blocked"]), n
        yb = po.conv_oracle64_blocked(g[f"{n}/x_blocked"], g[f"{n}/k_blocked"], ci, co, s)
        assert np.array_equal(yb, g[f"{n}/y_oracle64_blocked"]), n


def test_oracle_matches_live_reference():
    r = po.ref()
    if r is None:
        pytest.skip("reference sources not built here (GPU box)")
    F = ctypes.POINTER(ctypes.c_float)
    rng = np.random.default_rng(11)
    for t in range(12):
        ci, co = (int(v) for v in rng.integers(1, 12, 2))
        hf, wf = (int(v) for v in rng.choice([1, 2, 3, 5], 2))
        s = int(rng.choice([1, 2, 3]))
        ho, wo = (int(v) for v in rng.integers(1, 6, 2))
        hi, wi = (ho - 1) * s + hf, (wo - 1) * s + wf
        x = po.uniform((ci, hi, wi), 12, t)
        k = po.uniform((ci, co, hf, wf), 13, t)
        o = np.empty((co, ho, wo), np.float32)
        assert r.ref_conv(0, x.ctypes.data_as(F), k.ctypes.data_as(F), ci, co, hi, wi,
                          hf, wf, s, o.ctypes.data_as(F)) == 0
        assert np.array_equal(po.conv_oracle64(x, k, s), o)


def test_conv_direct_restatement_spec_cases(golden):
    """Restated Alg. 3 (the CPU baseline) vs the reference oracle."""
    g, names = golden
    for n in names:
        ci, co, hi, wi, hf, wf, s, cib, cob = g[f"{n}/geom"].tolist()
        for w_ob in (1, 3, 4):
            y = po.conv_direct(g[f"{n}/x_blocked"], g[f"{n}/k_blocked"], ci, co, s, w_ob=w_ob)
            ok, nbad, err = po.within_tol(y, g[f"{n}/y_oracle64_blocked"])
            assert ok, (n, w_ob, nbad, err)
    # 1x1x1 trivial -> 6
    y = po.conv_direct(np.array([[[[2.0]]]], np.float32),
                       np.array([[[[[[3.0]]]]]], np.float32), 1, 1, 1, w_ob=1)
    assert y.item() == 6.0


def test_conv_direct_thread_determinism():
    """SPEC.md:348 / acceptance 4: bitwise equal for any worker count."""
    x = po.pack_feature_map(po.uniform((16, 14, 14), 21, 0), 8)
    k = po.pack_kernel(po.uniform((16, 64, 3, 3), 21, 1), 8, 8)
    outs = [po.conv_direct(x, k, 16, 64, 1, threads=t) for t in (1, 2, 4, 8)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_mutation_literal_alg3_fails_on_stride2():
    """the literal PAPER.md:349 index must fail at s=2."""
    ci, co, hi, wi, hf, wf, s = 4, 8, 11, 11, 3, 3, 2
    x = po.uniform((ci, hi, wi), 31, 0)
    k = po.uniform((ci, co, hf, wf), 31, 1)
    xb, kb = po.pack_feature_map(x, 4), po.pack_kernel(k, 8, 4)
    want = po.pack_feature_map(po.conv_oracle64(x, k, s), 8)
    ho, wo = po.conv_shape(ci, co, hi, wi, hf, wf, s)
    out = np.empty_like(want)
    F = ctypes.POINTER(ctypes.c_float)
    assert po.orc().orc_conv_direct_literal_alg3(
        xb.ctypes.data_as(F), kb.ctypes.data_as(F), ci, co, hi, wi, hf, wf, s, 4, 8, 2,
        out.ctypes.data_as(F)) == 0
    assert not po.within_tol(out, want)[0]
    fixed = po.conv_direct(xb, kb, ci, co, s, w_ob=2)
    assert po.within_tol(fixed, want)[0]


def test_relu_add_pool_oracles():
    x = np.array([-1.0, 0.0, 2.0], np.float32)
    po.orc().orc_relu(x.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 3)
    assert x.tolist() == [0.0, 0.0, 2.0]
    a = po.uniform((2, 4, 6, 8), 41, 0)
    o = np.empty((2, 2, 3, 8), np.float32)
    po.orc().orc_maxpool2x2(a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 2, 4, 6, 8,
                            o.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    want = a.reshape(2, 2, 2, 3, 2, 8).max(axis=(2, 4))
    assert np.array_equal(o, want)


def test_uniform_generator_deterministic():
    a = po.uniform((1000,), 5, 3)
    b = po.uniform((1000,), 5, 3)
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0
    assert not np.array_equal(a, po.uniform((1000,), 5, 4))
