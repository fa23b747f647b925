"""GPU parity of the segmented (CSR) front end vs the oracle (BASELINE cfg4).

Segments of length <= 16 use the exact-length network (DAG-exact in REF mode),
longer ones the warp RSS sorter; empty and single-item segments are no-ops.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _csr(lengths):
    off = np.zeros(len(lengths) + 1, dtype=np.uint32)
    np.cumsum(lengths, out=off[1:])
    return off


def _run(torch, off, keys, pay, **kw):
    from paper_2002_05599_b200 import batch
    dev = torch.device("cuda")
    ot = torch.from_numpy(off.view(np.int32)).to(dev).view(torch.uint32)
    kt = torch.from_numpy(keys).to(dev) if keys.dtype.kind != "u" else \
        torch.from_numpy(keys.view(np.int32 if keys.dtype.itemsize == 4 else np.int64)).to(dev).view(
            torch.uint32 if keys.dtype.itemsize == 4 else torch.uint64)
    pt = None
    if pay is not None:
        pt = torch.from_numpy(pay.view(np.int32 if pay.dtype.itemsize == 4 else np.int64)).to(dev).view(
            torch.uint32 if pay.dtype.itemsize == 4 else torch.uint64)
    k, p = batch.sort_segments(ot, kt, pt, **kw)
    k = k.cpu().numpy().view(keys.dtype)
    p = p.cpu().numpy().view(pay.dtype) if pay is not None else None
    return k, p


def test_cfg4_shape_small_vs_oracle(torch):
    """cfg4 in miniature: f32 weights in [0,1) + u32 ids, descending by (w, id)."""
    nseg = 300_000
    lengths = oracle.geometric_lengths(nseg, seed=4)
    off = _csr(lengths)
    e = int(off[-1])
    u = oracle.splitmix(e, seed=40)
    w = ((u >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)
    ids = (u & np.uint64((1 << 26) - 1)).astype(np.uint32)
    w[1::2] = w[0::2][: len(w[1::2])]  # force weight ties inside segments
    for family in ("best", "bn-l"):
        for tie in ("unique", "ref"):
            ek, ep = oracle.typed_sort_segments(off, w, ids, family=family, descending=True,
                                                unique=tie == "unique")
            gk, gp = _run(torch, off, w, ids, family=family, descending=True, tie=tie)
            assert np.array_equal(gk.view(np.uint32), ek.view(np.uint32)), (family, tie)
            assert np.array_equal(gp, ep), (family, tie)
    # UNIQUE mode equals lexsort descending by (w, id) per segment
    gk, gp = _run(torch, off, w, ids, descending=True, tie="unique")
    for s in range(0, nseg, 997):
        a, b = off[s], off[s + 1]
        o = np.lexsort((ids[a:b], w[a:b]))[::-1]
        assert np.array_equal(gk[a:b], w[a:b][o]) and np.array_equal(gp[a:b], ids[a:b][o])


@pytest.mark.parametrize("kdt", ["uint32", "uint64", "int64", "float32"])
@pytest.mark.parametrize("pdt", [None, "uint32", "uint64"])
def test_segments_edge_lengths_vs_oracle(kdt, pdt, torch):
    rng = np.random.default_rng(8)
    lengths = np.concatenate([np.zeros(50, np.uint32), np.ones(50, np.uint32),
                              np.arange(0, 40, dtype=np.uint32), rng.integers(0, 17, 5000).astype(np.uint32),
                              np.array([1024, 17, 300, 0, 16, 1000], dtype=np.uint32)])
    rng.shuffle(lengths)
    off = _csr(lengths)
    e = int(off[-1])
    if kdt.startswith("float"):
        keys = np.round(rng.standard_normal(e) * 3).astype(kdt)
    else:
        keys = rng.integers(0, 6, size=e).astype(kdt)
    pay = None if pdt is None else rng.integers(0, 2**31, size=e).astype(pdt)
    for tie in (["unique"] if pdt is None else ["unique", "ref"]):
        for desc in (False, True):
            ek, ep = oracle.typed_sort_segments(off, keys, pay, descending=desc, unique=tie == "unique")
            gk, gp = _run(torch, off, keys, pay, descending=desc, tie=tie)
            assert np.array_equal(gk.view(np.uint8), ek.view(np.uint8)), (tie, desc)
            if pay is not None:
                assert np.array_equal(gp, ep), (tie, desc)


def test_segments_tile_overflow_split(torch):
    # 1024 segments of 16 items = 16384 items per tile > staging capacity: split path
    lengths = np.full(5000, 16, dtype=np.uint32)
    off = _csr(lengths)
    rng = np.random.default_rng(1)
    keys = rng.integers(0, 2**64, size=int(off[-1]), dtype=np.uint64)
    pay = np.arange(int(off[-1]), dtype=np.uint64)
    ek, ep = oracle.typed_sort_segments(off, keys, pay, unique=True)
    gk, gp = _run(torch, off, keys, pay, tie="unique")
    assert np.array_equal(gk, ek) and np.array_equal(gp, ep)


@pytest.mark.parametrize("tie", ["unique", "ref"])
def test_segments_pipeline_transitions(tie, torch):
    """More tiles than CTAs, so every CTA walks several tiles and the
    software pipeline (count tile k+1 while tile k sorts) runs; stretches of
    16-item segments make some tiles exceed the staging buffer, so the kernel
    moves between pipelined tiles and synchronous sub-tiles.  Whole output
    against the oracle, float weights descending with ties."""
    rng = np.random.default_rng(77)
    nseg = 1_300_000
    lengths = oracle.geometric_lengths(nseg, seed=9).astype(np.uint32)
    for lo in rng.integers(0, nseg - 5000, 120):
        lengths[lo:lo + int(rng.integers(200, 4000))] = 16
    lengths[rng.integers(0, nseg, 50)] = rng.integers(17, 300, 50).astype(np.uint32)
    off = _csr(lengths)
    e = int(off[-1])
    w = (rng.integers(-40, 40, e) / 8.0).astype(np.float32)
    w[rng.integers(0, e, 1000)] = -0.0
    ids = rng.integers(0, 1 << 26, e).astype(np.uint32)
    ek, ep = oracle.typed_sort_segments(off, w, ids, descending=True, unique=tie == "unique")
    gk, gp = _run(torch, off, w, ids, descending=True, tie=tie)
    assert np.array_equal(gk.view(np.uint32), ek.view(np.uint32))
    assert np.array_equal(gp, ep)


def test_cfg4_full_size_properties(torch):
    """cfg4 at full size: 67,108,864 segments; every segment sorted descending
    by (w, id) and a permutation of its input (checked on the device)."""
    from paper_2002_05599_b200 import batch
    nseg = 67_108_864
    dev = torch.device("cuda")
    lengths = oracle.geometric_lengths(nseg, seed=4)
    off = _csr(lengths)
    e = int(off[-1])
    u = oracle.splitmix(e, seed=40)
    w = ((u >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)
    ids = (u & np.uint64((1 << 26) - 1)).astype(np.uint32)
    ot = torch.from_numpy(off.view(np.int32)).to(dev).view(torch.uint32)
    wt = torch.from_numpy(w).to(dev)
    it = torch.from_numpy(ids.view(np.int32)).to(dev).view(torch.uint32)
    gk, gp = batch.sort_segments(ot, wt, it, descending=True, tie="unique")
    torch.cuda.synchronize()
    # composite key (w bits << 32 | id) must be non-increasing inside each segment
    comp = (gk.view(torch.int32).to(torch.int64) << 32) | gp.view(torch.int32).to(torch.int64).bitwise_and(0xFFFFFFFF)
    seg_of = torch.repeat_interleave(torch.arange(nseg, device=dev), torch.from_numpy(lengths.astype(np.int64)).to(dev))
    same = seg_of[1:] == seg_of[:-1]
    assert bool((comp[1:][same] <= comp[:-1][same]).all())
    comp_in = (wt.view(torch.int32).to(torch.int64) << 32) | it.view(torch.int32).to(torch.int64).bitwise_and(0xFFFFFFFF)
    # multiset per segment: sum and sum of squares (mod 2^64) of composite keys
    s_in = torch.zeros(nseg, dtype=torch.int64, device=dev).index_add_(0, seg_of, comp_in)
    s_out = torch.zeros(nseg, dtype=torch.int64, device=dev).index_add_(0, seg_of, comp)
    assert torch.equal(s_in, s_out)
    x_in = torch.zeros(nseg, dtype=torch.int64, device=dev).index_add_(0, seg_of, comp_in * comp_in)
    x_out = torch.zeros(nseg, dtype=torch.int64, device=dev).index_add_(0, seg_of, comp * comp)
    assert torch.equal(x_in, x_out)
    # a sampled window against the oracle
    lo, hi = 1_000_000, 1_050_000
    sub_off = (off[lo:hi + 1] - off[lo]).astype(np.uint32)
    ek, ep = oracle.typed_sort_segments(sub_off, w[off[lo]:off[hi]], ids[off[lo]:off[hi]], descending=True)
    assert np.array_equal(gk[off[lo]:off[hi]].cpu().numpy(), ek)
    assert np.array_equal(gp[off[lo]:off[hi]].cpu().numpy().view(np.uint32), ep)


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_segments_unaligned_offsets(shift, torch):
    """An offsets array that is not 16-byte aligned (a view into a larger
    buffer) takes the 4-byte copy path; the aligned path zero-fills its last
    16-byte chunk -- both must give the oracle's result."""
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(20 + shift)
    nseg = 4099 + shift
    lengths = rng.integers(0, 14, nseg).astype(np.uint32)
    off = _csr(lengths)
    e = int(off[-1])
    keys = rng.integers(0, 50, e).astype(np.uint32)
    pay = np.arange(e, dtype=np.uint32)
    dev = torch.device("cuda")
    buf = torch.zeros(len(off) + shift, dtype=torch.int32, device=dev)
    buf[shift:] = torch.from_numpy(off.view(np.int32)).to(dev)
    ot = buf[shift:].view(torch.uint32)
    assert ot.data_ptr() % 16 != 0
    kt = torch.from_numpy(keys.view(np.int32)).to(dev).view(torch.uint32)
    pt = torch.from_numpy(pay.view(np.int32)).to(dev).view(torch.uint32)
    gk, gp = batch.sort_segments(ot, kt, pt, tie="unique")
    ek, ep = oracle.typed_sort_segments(off, keys, pay, unique=True)
    assert np.array_equal(gk.cpu().numpy().view(np.uint32), ek)
    assert np.array_equal(gp.cpu().numpy().view(np.uint32), ep)


def test_segments_longer_than_1024(torch):
    """Keys-only / UNIQUE segments above 1024 items go to the CTA sorter
    (csrc/bigsort.cu) up to its shared-memory capacity; REF mode with a
    payload stops at 1024 and beyond-capacity segments fail loudly
    (nsg_segments_check) instead of returning unsorted data."""
    from paper_2002_05599_b200.errors import ConfigurationError
    rng = np.random.default_rng(1025)
    lengths = np.array([5, 1025, 3, 0, 20000, 1, 4096, 17, 1024], dtype=np.uint32)
    off = _csr(lengths)
    keys = rng.integers(0, 2**32, size=int(off[-1]), dtype=np.uint64).astype(np.uint32)
    keys[::3] %= 11
    gk, _ = _run(torch, off, keys, None)
    ek, _ = oracle.typed_sort_segments(off, keys, None)
    assert np.array_equal(gk, ek)
    off = _csr(np.array([5, 1025, 3, 0, 9000, 1, 4096, 17, 1024], dtype=np.uint32))  # <= 16384 8-byte items
    keys = keys[: int(off[-1])].copy()
    pay = rng.integers(0, 2**32, size=int(off[-1]), dtype=np.uint64).astype(np.uint32)
    for desc in (False, True):
        gk, gp = _run(torch, off, keys, pay, tie="unique", descending=desc)
        ek, ep = oracle.typed_sort_segments(off, keys, pay, unique=True, descending=desc)
        assert np.array_equal(gk, ek) and np.array_equal(gp, ep), desc
    # REF mode with a payload: the reference's tie order is replayed up to 1024
    with pytest.raises(ConfigurationError, match="device limit"):
        _run(torch, _csr(np.array([5, 1025, 3], dtype=np.uint32)),
             np.arange(1033, dtype=np.uint32)[::-1].copy(), np.arange(1033, dtype=np.uint32), tie="ref")
    # above the CTA sorter's shared-memory capacity (32768 4-byte keys)
    off = _csr(np.array([5, 40000, 3], dtype=np.uint32))
    with pytest.raises(ConfigurationError, match="device limit"):
        _run(torch, off, np.arange(int(off[-1]), dtype=np.uint32)[::-1].copy(), None)
