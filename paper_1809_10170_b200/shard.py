"""Multi-GPU partitioning of the direct-convolution path.

Two modes, one process per GPU (torch.distributed, NCCL over NVLink on the
box, gloo in the CPU tests):

* **Batch sharding** -- independent images.  Rank r owns the contiguous image
  range ``batch_range(N, P, r)``; weights are replicated; no collective on the
  data path (bench.py's default, weak in the sense that nothing is exchanged).

* **Output-block (C_o) sharding** -- batch 1.  Rank r owns the output blocks
  ``[r*B/P, (r+1)*B/P)`` with B = C_o/c_ob.  Because BlockedKernel is
  j'-outermost (tensor.hpp:131-140) a rank's weights are one contiguous slab
  range, and because a blocked map is block-outermost (tensor.hpp:71-74) a
  rank's output slice is one contiguous range too: the all-gather of equal
  slices *is* the full blocked map, with zero reshapes.  Element-wise work
  (ReLU, skip-add, max-pool) runs on the local slice before the gather.
"""
from __future__ import annotations

from typing import Tuple

import torch


def batch_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous image range [start, start+count) of ``rank``: sizes differ
    by at most one and the ranges tile [0, n) in rank order."""
    if not (0 <= rank < world) or n < 0:
        raise ValueError("batch_range: bad rank/world")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def block_range(n_blocks: int, world: int, rank: int) -> Tuple[int, int]:
    """Output blocks [begin, begin+count) of ``rank`` for C_o sharding.
    Equal slices are required for the all-gather: n_blocks % world == 0
    (choose c_ob <= C_o/P, e.g. c_ob = 8 gives 8 blocks for C_o = 64)."""
    if n_blocks % world:
        raise ValueError(f"C_o sharding needs blocks ({n_blocks}) divisible by ranks ({world})")
    per = n_blocks // world
    return rank * per, per


def weight_slab(w_blocked: torch.Tensor, begin: int, count: int) -> torch.Tensor:
    """Rank-local weights: the contiguous j' range of a blocked kernel
    [C_o/c_ob][C_i/c_ib][H_f][W_f][c_ib][c_ob] (a view, no copy)."""
    return w_blocked[begin:begin + count]


def all_gather_blocks(full: torch.Tensor, local: torch.Tensor, group=None) -> torch.Tensor:
    """Assemble the full blocked map from per-rank contiguous block slices.

    ``full``  : [B, ...] (B = world * local blocks), written in place
    ``local`` : [B/world, ...] this rank's slice (any block-outermost layout,
                halo ring included -- the ring is zero on every rank)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if full.shape[0] != world * local.shape[0] or full.shape[1:] != local.shape[1:]:
        raise ValueError("all_gather_blocks: layout error (slice shape)")
    if not (full.is_contiguous() and local.is_contiguous()):
        raise ValueError("all_gather_blocks: buffers must be contiguous")
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, local, group=group)
    else:  # gloo (CPU tests): list form, same result
        parts = list(full.chunk(world, dim=0))
        dist.all_gather(parts, local, group=group)
    return full
