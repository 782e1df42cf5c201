"""Generates tests/golden/golden.npz from the REFERENCE ITSELF.

Run here (where /root/reference exists) after `make -C oracle`: it calls the
reference's unmodified conv_oracle64 / conv_naive / conv_reordered /
pack_kernel / pack_feature_map (reference.cpp, tensor.cpp via
oracle/_ref/libdconv_ref.so) on seeded inputs and stores inputs and outputs.
The fixtures then pin oracle/oracle.c (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_parity.py) on machines without the reference.
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle as po  # noqa: E402

F = ctypes.POINTER(ctypes.c_float)


def fp(a):
    return a.ctypes.data_as(F)


# (name, c_i, c_o, h_i, w_i, h_f, w_f, s, c_ib, c_ob)
CASES = [
    ("spec_direct_8x16_12x12", 8, 16, 12, 12, 3, 3, 1, 8, 8),
    ("spec_direct_s2_4x8_11x11", 4, 8, 11, 11, 3, 3, 2, 4, 8),
    ("spec_edge_w7", 3, 6, 9, 9, 3, 3, 1, 4, 8),
    ("cfg1_small", 16, 16, 10, 10, 3, 3, 1, 8, 8),
    ("k5_s1", 12, 20, 13, 14, 5, 5, 1, 8, 8),
    ("k7_s2", 3, 16, 21, 21, 7, 7, 2, 3, 8),
    ("k11_s4", 3, 8, 27, 27, 11, 11, 4, 3, 8),
    ("k1_s2", 24, 16, 9, 9, 1, 1, 2, 8, 8),
    ("k3_s1_cb16", 32, 48, 9, 11, 3, 3, 1, 16, 16),
    ("odd_blocks", 5, 7, 6, 9, 2, 3, 2, 2, 4),
]


def main():
    ref = po.ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libdconv_ref.so not built")
    out = {}
    for idx, (name, ci, co, hi, wi, hf, wf, s, cib, cob) in enumerate(CASES):
        x = po.uniform((ci, hi, wi), 1809, 2 * idx)
        k = po.uniform((ci, co, hf, wf), 1809, 2 * idx + 1)
        ho, wo = po.conv_shape(ci, co, hi, wi, hf, wf, s)
        y = {}
        for mode, tag in ((0, "oracle64"), (1, "naive"), (2, "reordered")):
            o = np.empty((co, ho, wo), np.float32)
            assert ref.ref_conv(mode, fp(x), fp(k), ci, co, hi, wi, hf, wf, s, fp(o)) == 0
            y[tag] = o
        xb = np.zeros((po.round_up(ci, cib) // cib, hi, wi, cib), np.float32)
        ref.ref_pack_feature_map(fp(x), ci, hi, wi, cib, fp(xb))
        kb = np.zeros((po.round_up(co, cob) // cob, po.round_up(ci, cib) // cib, hf, wf, cib, cob),
                      np.float32)
        ref.ref_pack_kernel(fp(k), ci, co, hf, wf, cob, cib, fp(kb))
        yb = np.zeros((po.round_up(co, cob) // cob, ho, wo, cob), np.float32)
        ref.ref_pack_feature_map(fp(y["oracle64"]), co, ho, wo, cob, fp(yb))
        out[f"{name}/geom"] = np.array([ci, co, hi, wi, hf, wf, s, cib, cob], np.int64)
        out[f"{name}/x"] = x
        out[f"{name}/k"] = k
        out[f"{name}/x_blocked"] = xb
        out[f"{name}/k_blocked"] = kb
        out[f"{name}/y_oracle64_blocked"] = yb
        for tag, o in y.items():
            out[f"{name}/y_{tag}"] = o
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
