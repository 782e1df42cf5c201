"""Whole-output parity of the bench workloads at their full BASELINE batch
(VGG-16 b32, ResNet-50 b256, GoogLeNet b64), FFMA and split-TF32 plans:
EVERY element of EVERY conv launch is checked against the fp64 GPU referee
(oracle/oracle_gpu.cu, bit-exact with conv_oracle64, reference.cpp:70-87,
pinned by tests/test_oracle_gpu.py):

* chain: the plan runs as the bench runs it; each launch's output is compared
  with the referee on that launch's own (teacher-forced) input, normwise per
  layer: max|a-b| <= 1e-5 * max|want| + 1e-4 (deep unnormalised chains grow
  their activations);
* fresh inputs: each launch again, alone, on fresh uniform[-1,1) inputs (and
  skip tensors), per element at the fp32 tolerance |a-b| <= 1e-4 + 1e-5|b|.

Epilogues (ReLU, skip-add, fused 2x2 max-pool) are applied to the fp64
result before the comparison.  Slow (several TFLOP of fp64 on the GPU)."""
import numpy as np
import pytest
import torch

from oracle import gpu_oracle as go
from paper_1809_10170_b200 import _abi, nets

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _dense_weights(config: str, seed: int):
    """The dense [C_i][C_o][H_f][W_f] weights build_plan would generate."""
    ws = {}
    for idx, l in enumerate(nets.CONFIGS[config]):
        wd = torch.empty((l.c_i, l.c_o, l.h_f, l.w_f), dtype=torch.float32, device="cuda")
        scale = (3.0 / (l.c_i * l.h_f * l.w_f)) ** 0.5 if config == "resnet50" else 1.0
        nets._fill(wd, seed, 1000 + 2 * idx, scale)
        ws[l.name] = wd
    return ws


def _record(plan):
    """Run the plan once with spies on the conv launchers: per conv step,
    (layer, input Act / dense tensor, output Act, epilogue, skip Act,
    in_view).  Steps and launches pair up in order."""
    calls = []
    oc, ot = nets.conv, nets.conv_tf32

    def spy_c(l, n, x, w, out, epilogue=0, skip=None, stream=None, in_view=None, *a, **kw):
        oc(l, n, x, w, out, epilogue, skip, stream, in_view, *a, **kw)
        calls.append((x, out, epilogue, skip, in_view))

    def spy_t(l, n, x, wp, out, epilogue=0, skip=None, stream=None, in_view=None, **kw):
        ot(l, n, x, wp, out, epilogue, skip, stream, in_view, **kw)
        calls.append((x, out, epilogue, skip, in_view))
    nets.conv, nets.conv_tf32 = spy_c, spy_t
    try:
        plan.run()
    finally:
        nets.conv, nets.conv_tf32 = oc, ot
    torch.cuda.synchronize()
    convs = [(i, st) for i, st in enumerate(plan.steps) if st.kind in ("conv", "first", "tf32")]
    assert len(convs) == len(calls)
    return [(i, st, c) for (i, st), c in zip(convs, calls)]


def _want(plan, st, x, epilogue, skip, in_view, wd):
    """fp64 referee of one launch of layer st.layer (epilogue applied),
    blocked [n][jb][h][w][8] (pooled when the epilogue pools)."""
    l = st.layer
    if l.first:
        want = go.conv64_act(plan.input, l, wd)
    elif in_view is not None:
        ptr_, img, blk, row = in_view
        want = go.conv64(ptr_, plan.n, l.c_i, l.h_i, l.w_i, 8, img, blk, row, wd, l.s)
    else:
        want = go.conv64_act(x, l, wd)
    if epilogue & _abi.EPI_ADD:
        sk = skip.buf[:, :, skip.halo:skip.halo + l.h_o, skip.halo:skip.halo + l.w_o, :]
        want = want + sk.double()
    if epilogue & _abi.EPI_RELU:
        want = want.clamp_min(0.0)
    if epilogue & _abi.EPI_MAXPOOL:
        n, jb, h, w, c = want.shape
        want = want.view(n, jb, h // 2, 2, w // 2, 2, c).amax(dim=(3, 5))
    return want


def _got(out: nets.Act):
    return out.buf[:, :, out.halo:out.halo + out.h, out.halo:out.halo + out.w, :]


@pytest.mark.parametrize("algo", ["ffma", "tf32x3"])
@pytest.mark.parametrize("config,n", [("googlenet", 64), ("vgg16", 32), ("resnet50", 256)])
def test_every_element_every_layer(config, n, algo, monkeypatch):
    if algo == "tf32x3":
        # every blocked layer on the tensor cores (the bench batch has more
        # units than SMs anyway; keep the routing explicit)
        monkeypatch.setattr(nets.Plan, "_few_units", lambda self, l, epi: False)
    seed = 31
    wd = _dense_weights(config, seed)
    plan = nets.build_plan(config, n, seed=seed, dense_weights=wd, algo=algo)
    rec = _record(plan)
    checked = 0
    # (1) the chain as the bench runs it, teacher-forced, normwise per layer
    for i, st, (x, out, epi, skip, iv) in rec:
        want = _want(plan, st, x, epi, skip, iv, wd[st.layer.name]).float().double()
        got = _got(out).double()
        assert got.shape == want.shape, (st.name, got.shape, want.shape)
        scale = float(want.abs().max())
        err = float((got - want).abs().max())
        assert err <= 1e-5 * scale + 1e-4, f"{config}/{algo}/{st.name} chain: err {err} scale {scale}"
        checked += want.numel()
    # (2) every launch alone on fresh inputs, per element at the fp32 bound
    worst = 0.0
    for i, st, (x, out, epi, skip, iv) in rec:
        l = st.layer
        src = plan.input if l.first else x
        nets._fill(src if isinstance(src, torch.Tensor) else src.buf, 4000 + i, 1)
        if skip is not None:
            nets._fill(skip.buf, 5000 + i, 1)
        if l.first and i > 0 and plan.steps[i - 1].name == f"pack_{l.name}":
            plan.steps[i - 1].fn(None)  # the tensor-core stem's repack of the image
        st.fn(None)
        torch.cuda.synchronize()
        want = _want(plan, st, x, epi, skip, iv, wd[l.name])
        ok, nbad, err, ratio = go.check_tol(_got(out), want)
        assert ok, f"{config}/{algo}/{st.name} fresh: {nbad} elements out of tolerance, max err {err}"
        worst = max(worst, ratio)
    print(f"{config} b{n} {algo}: {len(rec)} launches, {checked} outputs (chain) + same "
          f"(fresh inputs); worst element at {worst:.3f} of the fp32 bound")
