"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic
of paper_1809_10170_b200/shard.py.  The per-rank compute is the CPU checker
(oracle.conv_direct, the restated Alg. 3), so what is tested is exactly the
partitioning / gather logic the GPU path uses with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po
from paper_1809_10170_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, msg in res.items():
        assert msg == "ok", f"rank {r}:\n{msg}"


# ------------------------------------------------------------------ bodies
def _batch_shard_body(rank, world):
    n, ci, co, hi, f, s = 5, 16, 24, 9, 3, 1
    xs = np.stack([po.pack_feature_map(po.uniform((ci, hi, hi), 11, i), 8) for i in range(n)])
    kb = po.pack_kernel(po.uniform((ci, co, f, f), 11, 99), 8, 8)
    start, cnt = shard.batch_range(n, world, rank)
    local = po.conv_direct(xs[start:start + cnt], kb, ci, co, s)
    # variable-size shards: gather as objects (test harness only)
    parts = [None] * world
    dist.all_gather_object(parts, (start, local))
    full = np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])])
    assert np.array_equal(full, po.conv_direct(xs, kb, ci, co, s))


def _co_shard_body(rank, world):
    ci, co, hi, f, s = 16, 32, 10, 3, 1
    x = po.pack_feature_map(po.uniform((ci, hi, hi), 21, 0), 8)
    kb = po.pack_kernel(po.uniform((ci, co, f, f), 21, 1), 8, 8)
    jb_n = kb.shape[0]
    b0, cnt = shard.block_range(jb_n, world, rank)
    wl = shard.weight_slab(torch.from_numpy(kb), b0, cnt).numpy()
    local = po.conv_direct(x, np.ascontiguousarray(wl), ci, cnt * 8, s)
    ho = hi - f + 1
    full = torch.zeros((jb_n, ho, ho, 8))
    shard.all_gather_blocks(full, torch.from_numpy(local))
    assert np.array_equal(full.numpy(), po.conv_direct(x, kb, ci, co, s))


def _co_shard_halo_chain_body(rank, world):
    """Two C_o-sharded layers: layer 1 writes (ReLU'd) into the interior of a
    halo'd slice, the gather yields the next layer's pre-padded input."""
    ci, c1, c2, h = 8, 16, 32, 7
    x = po.pack_feature_map(po.uniform((ci, h + 2, h + 2), 31, 0), 8)
    k1 = po.pack_kernel(po.uniform((ci, c1, 3, 3), 31, 1), 8, 8)
    k2 = po.pack_kernel(po.uniform((c1, c2, 3, 3), 31, 2), 8, 8)
    # layer 1 (3x3, 9 -> 7), output into a halo'd [blocks][9][9][8] buffer
    b0, cnt = shard.block_range(k1.shape[0], world, rank)
    y1 = np.maximum(po.conv_direct(x, np.ascontiguousarray(k1[b0:b0 + cnt]), ci, cnt * 8, 1), 0)
    local = torch.zeros((cnt, h + 2, h + 2, 8))
    local[:, 1:-1, 1:-1, :] = torch.from_numpy(y1)
    full1 = torch.zeros((k1.shape[0], h + 2, h + 2, 8))
    shard.all_gather_blocks(full1, local)
    # layer 2 on the gathered halo'd map
    b0, cnt = shard.block_range(k2.shape[0], world, rank)
    y2 = po.conv_direct(full1.numpy(), np.ascontiguousarray(k2[b0:b0 + cnt]), c1, cnt * 8, 1)
    full2 = torch.zeros((k2.shape[0], h, h, 8))
    shard.all_gather_blocks(full2, torch.from_numpy(y2))
    # unsharded reference
    r1 = np.maximum(po.conv_direct(x, k1, ci, c1, 1), 0)
    p1 = np.zeros((k1.shape[0], h + 2, h + 2, 8), np.float32)
    p1[:, 1:-1, 1:-1, :] = r1
    assert np.array_equal(full2.numpy(), po.conv_direct(p1, k2, c1, c2, 1))


# ------------------------------------------------------------------ tests
def test_batch_range_tiles_batch():
    for n in (0, 1, 5, 32, 256):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                s, c = shard.batch_range(n, world, r)
                covered += list(range(s, s + c))
            assert covered == list(range(n))


def test_block_range_contiguous_and_errors():
    assert [shard.block_range(8, 8, r) for r in range(8)] == [(r, 1) for r in range(8)]
    assert shard.block_range(256, 8, 3) == (96, 32)
    with pytest.raises(ValueError):
        shard.block_range(12, 8, 0)


def test_batch_sharding_gloo_world2():
    _run(_batch_shard_body)


def test_co_block_sharding_allgather_gloo_world2():
    _run(_co_shard_body)


def test_co_sharded_chain_with_halo_gloo_world2():
    _run(_co_shard_halo_chain_body)
