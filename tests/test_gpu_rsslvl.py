"""GPU parity of the packed-key RSS kernel (csrc/pksort.cu, PhaseRss) -- the
keys-only / UNIQUE path of `kind="rss"` for 17..256 items -- against the
oracle (reference restatement) and np.sort, including the inputs that force
its exact fallback (packed-key ties) and the reference RSS tests' shapes
(all-equal, presorted, duplicate-heavy rows: reference test_rss.py:208-254).
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

NS = (17, 20, 31, 32, 33, 50, 63, 64, 65, 100, 127, 128, 129, 200, 255, 256)


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _gen(rng, kind, m, n, dt=np.uint64):
    info = np.iinfo(dt)
    if kind == "uniform":
        return rng.integers(info.min, info.max, size=(m, n), dtype=dt, endpoint=True)
    if kind == "few":
        vals = rng.integers(info.min, info.max, size=16, dtype=dt, endpoint=True)
        return vals[rng.integers(0, 16, size=(m, n))]
    if kind == "dup":
        return rng.integers(0, 4, size=(m, n)).astype(dt)
    if kind == "sorted":
        return np.sort(rng.integers(info.min, info.max, size=(m, n), dtype=dt, endpoint=True), axis=1)
    if kind == "reverse":
        return np.sort(rng.integers(info.min, info.max, size=(m, n), dtype=dt, endpoint=True), axis=1)[:, ::-1].copy()
    if kind == "equal":
        return np.full((m, n), 12345, dtype=dt)
    if kind == "clustered":  # low-bit differences under a wide range: packed-key ties -> exact fallback
        base = np.array(1 << (8 * np.dtype(dt).itemsize - 2), dtype=dt)
        x = rng.integers(0, 1 << 12, size=(m, n)).astype(dt) + base
        x[:, 0] = 0  # widen the row so the kept prefix cannot see the low bits
        return x
    raise ValueError(kind)


def _sort(torch, keys, payload=None, **kw):
    from paper_2002_05599_b200 import batch
    kt = torch.from_numpy(keys.view(np.int64 if keys.dtype.itemsize == 8 else np.int32)).cuda()
    kt = kt.view({np.dtype(np.uint64): torch.uint64, np.dtype(np.int64): torch.int64,
                  np.dtype(np.uint32): torch.uint32, np.dtype(np.int32): torch.int32,
                  np.dtype(np.float32): torch.float32}[keys.dtype])
    pt = None
    if payload is not None:
        pt = torch.from_numpy(payload.view(np.int32)).cuda().view(torch.uint32)
    ok, op = batch.sort_rows(kt, pt, kind="rss", **kw)
    torch.cuda.synchronize()
    return ok.cpu().numpy(), (op.cpu().numpy() if op is not None else None)


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("dist", ["uniform", "few", "dup", "sorted", "reverse", "equal"])
def test_int64_keys_vs_np_sort(torch, n, dist):
    rng = np.random.default_rng(n * 131 + len(dist))
    keys = _gen(rng, dist, 1003, n, np.int64)  # 1003 rows: partial last warp group
    got, _ = _sort(torch, keys)
    assert np.array_equal(got, np.sort(keys, axis=1)), (n, dist)


@pytest.mark.parametrize("n", (24, 64, 100, 256))
def test_uint64_and_uint32_vs_oracle(torch, n):
    rng = np.random.default_rng(n)
    for dt in (np.uint64, np.uint32):
        keys = _gen(rng, "uniform", 700, n, dt)
        got, _ = _sort(torch, keys)
        ek, _ = oracle.typed_sort_rows(keys, kind="rss")
        assert np.array_equal(got, ek), (n, dt)


@pytest.mark.parametrize("n", (17, 96, 256))
def test_float32_descending_with_payload_unique(torch, n):
    rng = np.random.default_rng(7 + n)
    w = (rng.integers(0, 64, size=(500, n)) / 64.0).astype(np.float32)  # many weight ties
    ids = rng.integers(0, 1 << 26, size=(500, n)).astype(np.uint32)
    gk, gp = _sort(torch, w, ids, descending=True, tie="unique")
    ek, ep = oracle.typed_sort_rows(w, ids, descending=True, unique=True, kind="rss")
    assert np.array_equal(gk, ek) and np.array_equal(gp, ep)


@pytest.mark.parametrize("n", (40, 128, 256))
def test_u64_with_payload_unique_duplicate_heavy(torch, n):
    rng = np.random.default_rng(99 + n)
    keys = rng.integers(0, 8, size=(300, n)).astype(np.uint64)
    pay = rng.permutation(300 * n).astype(np.uint32).reshape(300, n)
    gk, gp = _sort(torch, keys, pay, tie="unique")
    ek, ep = oracle.typed_sort_rows(keys, pay, unique=True, kind="rss")
    assert np.array_equal(gk, ek) and np.array_equal(gp, ep)


@pytest.mark.parametrize("n", (33, 256))
def test_exact_fallback_rows(torch, n):
    """Rows whose keys differ only below the packed prefix go through the
    exact warp sorter; the result is still the unique sorted order."""
    from paper_2002_05599_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(5)
    keys = _gen(rng, "clustered", 400, n, np.uint64)
    lib.nsg_rss_fallback_rows(1)
    got, _ = _sort(torch, keys)
    assert np.array_equal(got, np.sort(keys, axis=1))
    assert lib.nsg_rss_fallback_rows(1) > 0


def test_uniform_rows_rarely_fall_back(torch):
    from paper_2002_05599_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(11)
    keys = _gen(rng, "uniform", 4096, 256, np.int64)
    lib.nsg_rss_fallback_rows(1)
    got, _ = _sort(torch, keys)
    assert np.array_equal(got, np.sort(keys, axis=1))
    assert lib.nsg_rss_fallback_rows(1) < 4096 // 50


def test_in_place(torch):
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(3)
    keys = _gen(rng, "clustered", 257, 200, np.uint64)  # includes fallback rows
    kt = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
    batch.sort_rows(kt, kind="rss", out_keys=kt)
    torch.cuda.synchronize()
    assert np.array_equal(kt.cpu().numpy(), np.sort(keys, axis=1))
