"""Batch-1 C_o-block sharding at world sizes 2, 4 and 8, with the
ranks emulated on one GPU (B200_PROFILING.md: with fewer GPUs than ranks,
run the ranks' work without kernels that wait on one another):

* gather_mode "emulate": every rank's launch of a layer -- its output-block
  range, hence the kernel configuration a real rank runs -- one after
  another into one full map, i.e. exactly what the NCCL all-gather of the
  ranks' slices assembles;
* gather_mode "emulate_peer": every rank keeps its own full copy of every
  map and its conv / first-layer / pool epilogues also store into all other
  ranks' copies (the fused peer-store gather, peers = local buffers).

Checked: all ranks' copies identical and bitwise equal to the emulated
all-gather map; every element of every layer against the fp64 referee
(teacher-forced normwise on the chain, per element on fresh inputs); the
network output against the unsharded plan (normwise: the split-K factor of
a C_o slice differs, so rounding differs)."""
import pytest
import torch

from oracle import gpu_oracle as go
from paper_1809_10170_b200 import nets

from test_gpu_fullsize import _dense_weights, _got, _record, _want

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("config", ["resnet50", "vgg16"])
def test_co_shard_emulated_ranks(config, world):
    seed = 6
    wd = _dense_weights(config, seed)
    ref = nets.build_plan(config, 1, seed=seed, dense_weights=wd)
    emu = nets.build_plan(config, 1, seed=seed, dense_weights=wd, shard=(0, world, None),
                          gather_mode="emulate")
    peer = nets.build_plan(config, 1, seed=seed, dense_weights=wd, shard=(0, world, None),
                           gather_mode="emulate_peer")
    # every conv layer is split into `world` launches with disjoint block ranges
    assert sum(st.kind in ("conv", "first") for st in emu.steps) == world * len(emu.layers)
    ref.run()
    peer.run()
    rec = _record(emu)  # runs the emulated plan once
    torch.cuda.synchronize()
    # (a) fused peer gather: every rank's copy == the all-gather map, bitwise
    for name, a in emu.outputs.items():
        copies = peer.outputs[name].copies
        assert len(copies) == world
        for r, c in enumerate(copies):
            assert torch.equal(c.buf, a.buf), f"{name}: rank {r}'s copy differs"
    # (b) network output vs the unsharded plan
    want, got = ref.output.buf.double(), emu.output.buf.double()
    scale = float(want.abs().max())
    assert float((got - want).abs().max()) <= 1e-4 * max(1.0, scale)
    # (c) every element of every layer: teacher-forced (normwise) ...
    by_layer = {}
    for i, st, c in rec:
        by_layer.setdefault(st.layer.name, []).append((i, st, c))
    for name, launches in by_layer.items():
        i, st, (x, out, epi, skip, iv) = launches[0]
        w64 = _want(emu, st, x, epi, skip, iv, wd[name]).float().double()
        g = _got(_full_map(out, st.layer)).double()  # the map every rank's view wrote
        sc = float(w64.abs().max())
        assert float((g - w64).abs().max()) <= 1e-5 * sc + 1e-4, f"{config} w{world} {name}"
    # ... and per element on fresh inputs (all ranks' launches of a layer)
    for name, launches in by_layer.items():
        i, st, (x, out, epi, skip, iv) = launches[0]
        l = st.layer
        src = emu.input if l.first else x
        nets._fill(src if isinstance(src, torch.Tensor) else src.buf, 700 + i, 1)
        if skip is not None:
            nets._fill(skip.buf, 800 + i, 1)
        for j, stj, _ in launches:
            stj.fn(None)
        torch.cuda.synchronize()
        w64 = _want(emu, st, x, epi, skip, iv, wd[name])
        ok, nbad, err, ratio = go.check_tol(_got(_full_map(out, l)), w64)
        assert ok, f"{config} world {world} {name} fresh: {nbad} bad, max err {err}"


def _full_map(view: nets.Act, l) -> nets.Act:
    """The whole map behind a rank's block view (the views share the buffer;
    the interior origin of block 0 is the halo offset)."""
    import copy
    m = copy.copy(view)
    m.off = (m.halo * m.wp + m.halo) * nets.CB
    m.c = l.c_o
    return m
