"""Tensor files and weight ingest: the 7-int header +
little-endian fp32 format of SPEC.md:129 and the CLI `pack` step of
SPEC.md:580-587 ("pack then unpack file roundtrip -> byte-identical dense
kernel payload", "1-weight kernel file -> 1-weight packed file plus header",
"packing a file twice -> error 'already blocked'", "malformed file -> parse
error").  Header/parse/error paths run on the CPU; the GPU repack is
checked bit-exact against the oracle's pack_kernel."""
import os

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_1809_10170_b200 import _abi
from paper_1809_10170_b200 import dconv as D


def _blocked_file(path, k, cob, cib):
    ci, co, hf, wf = k.shape
    D._write(path, (ci, hf, wf, cob, co, cib, _abi.FILE_KERNEL), po.pack_kernel(k, cob, cib))


def test_header_roundtrip_and_payload(tmp_path):
    k = po.uniform((3, 5, 2, 2), 1, 2)
    p = str(tmp_path / "k.bin")
    D.save_kernel(p, k)
    assert os.path.getsize(p) == 28 + k.size * 4  # 7 int32 words + payload
    h, payload = D.read_payload(p)
    assert (h.c, h.h, h.w, h.c_b, h.c_o, h.c_ib, h.kind) == (3, 2, 2, 0, 5, 0, 1)
    assert payload.tobytes() == k.tobytes()
    raw = open(p, "rb").read()
    assert np.frombuffer(raw[:28], "<i4").tolist() == [3, 2, 2, 0, 5, 0, 1]
    assert np.frombuffer(raw[28:], "<f4").tobytes() == k.tobytes()


def test_feature_map_file_sizes(tmp_path):
    x = po.uniform((5, 4, 3), 2, 0)
    p = str(tmp_path / "x.bin")
    D.save_feature_map(p, x)
    h, payload = D.read_payload(p)
    assert (h.c, h.h, h.w, h.c_b, h.kind) == (5, 4, 3, 0, 0)
    assert np.array_equal(payload.reshape(x.shape), x)
    # blocked: payload covers the zero-padded channels
    D._write(p, (5, 4, 3, 8, 0, 0, _abi.FILE_FEATURE_MAP), po.pack_feature_map(x, 8))
    h, payload = D.read_payload(p)
    assert h.c_b == 8 and payload.size == 8 * 4 * 3


def test_malformed_files_are_parse_errors(tmp_path):
    p = str(tmp_path / "bad.bin")
    open(p, "wb").write(b"\x01\x00")
    with pytest.raises(ValueError, match="parse error"):
        D.read_header(p)
    # truncated payload
    k = po.uniform((2, 2, 1, 1), 3, 0)
    D.save_kernel(p, k)
    open(p, "r+b").truncate(28 + 8)
    with pytest.raises(ValueError, match="parse error"):
        D.read_header(p)
    # invalid header words (kernel with blocked c_ob but dense c_ib)
    open(p, "wb").write(np.array([2, 1, 1, 8, 2, 0, 1], "<i4").tobytes() + b"\0" * 64)
    with pytest.raises(ValueError, match="parse error"):
        D.read_header(p)
    # unknown kind
    open(p, "wb").write(np.array([1, 1, 1, 0, 0, 0, 9], "<i4").tobytes() + b"\0" * 4)
    with pytest.raises(ValueError, match="parse error"):
        D.read_header(p)
    with pytest.raises(_abi.DconvError, match="I/O"):
        D.read_header(str(tmp_path / "missing.bin"))


def test_packing_twice_is_already_blocked(tmp_path):
    k = po.uniform((4, 6, 3, 3), 4, 0)
    p = str(tmp_path / "kb.bin")
    _blocked_file(p, k, 8, 8)
    with pytest.raises(ValueError, match="already blocked"):
        D.pack_kernel_file(p, 8, 8, str(tmp_path / "again.bin"))
    assert not os.path.exists(tmp_path / "again.bin")


def test_pack_rejects_feature_map_files(tmp_path):
    p = str(tmp_path / "x.bin")
    D.save_feature_map(p, po.uniform((2, 2, 2), 5, 0))
    with pytest.raises(ValueError, match="not a kernel file"):
        D.pack_kernel_file(p, 8, 8, str(tmp_path / "o.bin"))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,cob,cib", [((5, 11, 3, 3), 8, 8), ((3, 64, 7, 7), 8, 3),
                                           ((1, 1, 1, 1), 8, 8), ((16, 24, 1, 1), 4, 16)])
def test_pack_file_roundtrip_bit_exact(tmp_path, shape, cob, cib):
    k = po.uniform(shape, 6, cob * 100 + cib)
    dense, blk, back = (str(tmp_path / n) for n in ("k.bin", "kb.bin", "kd.bin"))
    D.save_kernel(dense, k)
    D.pack_kernel_file(dense, cob, cib, blk)
    h, payload = D.read_payload(blk)
    assert (h.c_b, h.c_ib, h.c_o, h.c) == (cob, cib, shape[1], shape[0])
    assert payload.tobytes() == po.pack_kernel(k, cob, cib).tobytes()
    # unpack the ingested kernel on the GPU -> identical dense payload
    kb = D.load_kernel_file(blk, cob, cib)
    D.save_kernel(back, D.unpack_kernel(kb))
    assert open(back, "rb").read() == open(dense, "rb").read()


@pytest.mark.gpu
def test_ingest_dense_and_blocked_files(tmp_path):
    k = po.uniform((24, 40, 3, 3), 7, 0)
    dense, blk = str(tmp_path / "k.bin"), str(tmp_path / "kb.bin")
    D.save_kernel(dense, k)
    _blocked_file(blk, k, 8, 8)
    want = po.pack_kernel(k, 8, 8)
    for p in (dense, blk):
        got = D.load_kernel_file(p, 8, 8).data
        torch.cuda.synchronize()
        assert got.cpu().numpy().tobytes() == want.tobytes()
    with pytest.raises(ValueError, match="layout error"):
        D.load_kernel_file(blk, 4, 8)  # blocked with other block sizes
