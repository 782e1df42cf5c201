"""FFMA throughput at channel blocks c_b = 8 / 16 / 32 (c_ib = c_ob) on
representative layers (VGG-16 b32 and ResNet-50 b256 shapes), each CTA tile
timed (CUDA events, median of 5 after warm-up), best tile reported.
usage: python tools/cb_sweep.py [out.json]"""
import ctypes
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_10170_b200 import _abi  # noqa: E402
from paper_1809_10170_b200._abi import check, lib  # noqa: E402

LAYERS = [  # name, c_i, c_o, h_i, f, s, n
    ("vgg conv1_2 64->64 3x3 226", 64, 64, 226, 3, 1, 32),
    ("vgg conv3_2 256->256 3x3 58", 256, 256, 58, 3, 1, 32),
    ("vgg conv4_2 512->512 3x3 30", 512, 512, 30, 3, 1, 32),
    ("vgg conv5_2 512->512 3x3 16", 512, 512, 16, 3, 1, 32),
    ("resnet 1024->256 1x1 14", 1024, 256, 14, 1, 1, 256),
    ("resnet 256->1024 1x1 14", 256, 1024, 14, 1, 1, 256),
    ("resnet 128->128 3x3 30", 128, 128, 30, 3, 1, 256),
]


def time_layer(ci, co, hi, f, s, n, cb, tv):
    ho = (hi - f) // s + 1
    x = torch.empty((n, -(-ci // cb), hi, hi, cb), device="cuda").uniform_(-1, 1)
    w = torch.empty((-(-co // cb), -(-ci // cb), f, f, cb, cb), device="cuda").uniform_(-1, 1)
    y = torch.empty((n, -(-co // cb), ho, ho, cb), device="cuda")
    d = _abi.ConvDesc()
    check(lib().dconv_conv_desc_init(ctypes.byref(d), n, ci, co, hi, hi, f, f, s, cb, cb))
    d.algo, d.tile_variant, d.epilogue = _abi.ALGO_FFMA, tv, _abi.EPI_RELU
    st = torch.cuda.current_stream()

    def run():
        check(lib().dconv_cuda_conv_direct(ctypes.byref(d), x.data_ptr(), w.data_ptr(), 0,
                                           y.data_ptr(), st.cuda_stream))
    for _ in range(3):
        run()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    return 2 * ci * co * ho * ho * f * f * n / (ms * 1e-3) / 1e12, ms


def main():
    out = []
    for name, ci, co, hi, f, s, n in LAYERS:
        rec = {"layer": name}
        for cb in (8, 16, 32):
            best = max((time_layer(ci, co, hi, f, s, n, cb, tv) + (tv,) for tv in (1, 2)),
                       key=lambda t: t[0])
            rec[f"cb{cb}"] = {"tflops": round(best[0], 2), "ms": round(best[1], 4),
                              "tile": ["", "128x128", "256x64"][best[2]]}
        rec["cb16_vs_cb8"] = round(rec["cb16"]["tflops"] / rec["cb8"]["tflops"], 3)
        rec["cb32_vs_cb8"] = round(rec["cb32"]["tflops"] / rec["cb8"]["tflops"], 3)
        print(json.dumps(rec), flush=True)
        out.append(rec)
    if len(sys.argv) > 1:
        json.dump({"device": torch.cuda.get_device_name(0), "layers": out}, open(sys.argv[1], "w"),
                  indent=1)


if __name__ == "__main__":
    main()
