"""Multi-GPU sharding of independent batches (no data-path collective).

The arrays of a batch are independent, so N GPUs (one process per GPU,
torch.distributed for plumbing only) each sort a contiguous range:

  * fixed-width rows: rank r owns rows [r*B/N, (r+1)*B/N);
  * CSR segments: rank r owns a contiguous segment range whose ELEMENT count is
    balanced (split points found by binary search on the offsets); each shard
    rebases its offsets to start at 0;
  * synthetic inputs are generated from the GLOBAL element index, so the
    concatenation of the shards' outputs is bit-identical to a 1-GPU run.

The only collective is the timing reduction (max over ranks) and optional
result gathering in tests.
"""

from __future__ import annotations

import numpy as np


def shard_rows(total: int, rank: int, world: int) -> tuple:
    """Contiguous, balanced [lo, hi) row range of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return total * rank // world, total * (rank + 1) // world


def shard_segments(offsets: np.ndarray, rank: int, world: int) -> tuple:
    """(seg_lo, seg_hi) so every rank gets ~E/world elements, whole segments only."""
    offsets = np.asarray(offsets)
    nseg = len(offsets) - 1
    e = int(offsets[-1]) - int(offsets[0])

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return nseg
        target = int(offsets[0]) + e * r // world
        return int(np.searchsorted(offsets[:-1], target, side="left"))

    return cut(rank), cut(rank + 1)


def rebase_offsets(offsets: np.ndarray, seg_lo: int, seg_hi: int) -> tuple:
    """Local offsets (starting at 0) and the global element range of a shard."""
    off = np.asarray(offsets)[seg_lo:seg_hi + 1].astype(np.int64)
    e_lo, e_hi = int(off[0]), int(off[-1])
    return (off - e_lo).astype(np.uint32), e_lo, e_hi


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing over the process group (1 rank: identity)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
