"""N>1 host logic on CPU: world_size-2 gloo process group (no GPU needed).

Each rank sorts its contiguous shard (generated from the GLOBAL element
index) with the CPU oracle standing in for its GPU; the shards, gathered,
must equal a single-process run bit for bit, and the timing reduction must be
the max over ranks.  Mirrors bench.py's multi-GPU path and shard.py.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import oracle
        from paper_2002_05599_b200 import shard
        # fixed-width rows (cfg2 shape, small)
        total, n = 10_001, 9
        lo, hi = shard.shard_rows(total, rank, world)
        keys = oracle.splitmix((hi - lo) * n, seed=77, first=lo * n).reshape(hi - lo, n)
        pay = np.broadcast_to(np.arange(n, dtype=np.uint32), keys.shape).copy()
        k, p = oracle.typed_sort_rows(keys, pay, family="best", unique=True)
        kt = [torch.zeros(0)] * world
        dist.all_gather_object(kt, (lo, hi, k, p))
        # CSR segments balanced by elements
        lengths = oracle.geometric_lengths(5000, seed=3)
        off = np.zeros(5001, dtype=np.uint32)
        np.cumsum(lengths, out=off[1:])
        w = oracle.splitmix(int(off[-1]), seed=9, elem_bytes=4)
        s_lo, s_hi = shard.shard_segments(off, rank, world)
        loc, e_lo, e_hi = shard.rebase_offsets(off, s_lo, s_hi)
        sk, _ = oracle.typed_sort_segments(loc, w[e_lo:e_hi], None, descending=True)
        seg = [None] * world
        dist.all_gather_object(seg, (s_lo, s_hi, e_lo, e_hi, sk))
        t = shard.max_over_ranks(1.0 + rank)
        q.put((rank, kt, seg, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_equal_single_process():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # timing reduction = max over ranks
    assert all(r[3] == 2.0 for r in res)
    # rows: gathered shards == single run
    shards = res[0][1]
    assert shards[0][0] == 0 and shards[-1][1] == 10_001 and shards[0][1] == shards[1][0]
    k = np.concatenate([s[2] for s in shards])
    p = np.concatenate([s[3] for s in shards])
    full = oracle.splitmix(10_001 * 9, seed=77).reshape(10_001, 9)
    ek, ep = oracle.typed_sort_rows(full, np.broadcast_to(np.arange(9, dtype=np.uint32), full.shape).copy(),
                                    unique=True)
    assert np.array_equal(k, ek) and np.array_equal(p, ep)
    # segments: contiguous cover, balanced, equal to the single run
    segs = res[0][2]
    assert segs[0][0] == 0 and segs[-1][1] == 5000 and segs[0][1] == segs[1][0]
    lengths = oracle.geometric_lengths(5000, seed=3)
    off = np.zeros(5001, dtype=np.uint32)
    np.cumsum(lengths, out=off[1:])
    w = oracle.splitmix(int(off[-1]), seed=9, elem_bytes=4)
    ek, _ = oracle.typed_sort_segments(off, w, None, descending=True)
    assert np.array_equal(np.concatenate([s[4] for s in segs]), ek)
    sizes = [s[3] - s[2] for s in segs]
    assert abs(sizes[0] - sizes[1]) <= 32


def test_shard_helpers():
    from paper_2002_05599_b200 import shard
    for total in (0, 1, 7, 2**20 + 3):
        for world in (1, 2, 3, 8):
            rs = [shard.shard_rows(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        shard.shard_rows(10, 2, 2)
