"""CPU tests of the boundary: the C-ABI library loads without a GPU, exports
every symbol include/dconv_cuda.h declares, and its host-only entry points
(ConvShape validation, conv_flops, desc init) follow the reference's rules."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dconv_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dconv_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for s in ("dconv_cuda_conv_direct", "dconv_cuda_pack_kernel",
              "dconv_cuda_pack_feature_map", "dconv_cuda_relu_blocked",
              "dconv_cuda_conv_first_layer", "dconv_conv_shape"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1809_10170_b200 import _abi
    lib = _abi.lib()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(header_symbols()) == set(_abi.EXPORTED)


def test_host_only_entry_points():
    from paper_1809_10170_b200 import _abi
    from paper_1809_10170_b200.dconv import ConvShape, conv_flops
    s = ConvShape(64, 64, 58, 58, 3, 3, 1)
    assert (s.h_o, s.w_o) == (56, 56)
    assert conv_flops(ConvShape(3, 2, 4, 4, 2, 2)) == 432
    for bad in [(3, 64, 230, 230, 7, 7, 2), (1, 1, 2, 2, 3, 3, 1), (0, 1, 1, 1, 1, 1, 1),
                (1, 1, 5, 5, 1, 1, 0)]:
        with pytest.raises(ValueError, match="ConvShape"):
            ConvShape(*bad)
    d = _abi.ConvDesc()
    assert _abi.lib().dconv_conv_desc_init(ctypes.byref(d), 2, 3, 96, 227, 227, 11, 11, 4,
                                           3, 8) == 0
    assert (d.h_o, d.w_o, d.n) == (55, 55, 2)
    assert _abi.lib().dconv_conv_desc_init(ctypes.byref(d), 1, 3, 64, 230, 230, 7, 7, 2,
                                           8, 8) == _abi.EINVAL_SHAPE


def test_null_pointers_rejected_without_gpu():
    from paper_1809_10170_b200 import _abi
    lib = _abi.lib()
    d = _abi.ConvDesc()
    lib.dconv_conv_desc_init(ctypes.byref(d), 1, 8, 8, 5, 5, 3, 3, 1, 8, 8)
    assert lib.dconv_cuda_conv_direct(ctypes.byref(d), 0, 0, 0, 0, 0) == _abi.EPARAM
    assert lib.dconv_cuda_pack_kernel(0, 1, 1, 1, 1, 1, 1, 0, 0) == _abi.EPARAM
    d.epilogue = _abi.EPI_ADD
    assert lib.dconv_cuda_conv_direct(ctypes.byref(d), 16, 16, 0, 16, 0) == _abi.EPARAM


def test_product_package_never_imports_oracle():
    """The product path must not route through the CPU checker."""
    pkg = os.path.join(ROOT, "paper_1809_10170_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|pyoracle|"
                                     r"libdconv_ref|\borc_[a-z])", txt), f


def test_split_tf32_host_side():
    """Split-TF32 entry points on the host: the prepared buffer holds hi and
    lo halves (exactly twice the TF32 one), NULL arguments are refused
    before any launch, and the plan builder routes batch-1 layers with fewer
    tensor-core units than SMs to the FFMA kernel (same fp32 tolerance)."""
    from paper_1809_10170_b200 import _abi, nets
    lib = _abi.lib()
    for shp in [(64, 64, 58, 58, 3), (256, 1024, 14, 14, 1), (24, 40, 9, 9, 5)]:
        ci, co, h, w, f = shp
        d = _abi.ConvDesc()
        assert lib.dconv_conv_desc_init(ctypes.byref(d), 1, ci, co, h, w, f, f, 1, 8, 8) == 0
        a, b = ctypes.c_int64(0), ctypes.c_int64(0)
        assert lib.dconv_cuda_tf32_prepared_size(ctypes.byref(d), ctypes.byref(a)) == 0
        assert lib.dconv_cuda_tf32x3_prepared_size(ctypes.byref(d), ctypes.byref(b)) == 0
        assert b.value == 2 * a.value > 0
        assert lib.dconv_cuda_conv_direct_tf32x3(ctypes.byref(d), 0, 0, 0, 0, 0) == _abi.EPARAM
    assert lib.dconv_cuda_tf32x3_prepared_size(None, None) == _abi.EPARAM
    p = nets.Plan("t", 1, [], algo="tf32x3")
    assert p.x3 and "tf32x3" in nets.TC_ALGOS
    assert p._few_units(nets.Layer("c", 64, 64, 58, 58, 3, 3, 1), 0)       # cfg1 b1: 28 units
    assert not p._few_units(nets.Layer("c", 64, 64, 58, 58, 3, 3, 1), _abi.EPI_MAXPOOL)
    assert not nets.Plan("t", 32, [], algo="tf32x3")._few_units(
        nets.Layer("c", 64, 64, 58, 58, 3, 3, 1), 0)
