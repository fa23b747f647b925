"""GPU parity of the CTA sorter for rows and CSR segments above 1024 items
(csrc/bigsort.cu): keys-only and UNIQUE (key, payload) output
is the unique sorted order, so it must equal the reference-restating oracle
(RSS recursion, no size cap: netsort_core.c:325-391) and np.sort / lexsort,
both below the shared-memory capacity (one CTA bitonic sort) and above it
(tile sort + merge passes through a scratch copy)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _t(torch, x):
    x = np.ascontiguousarray(x)
    if x.dtype.kind == "u":
        sig = {4: np.int32, 8: np.int64}[x.dtype.itemsize]
        tdt = {4: torch.uint32, 8: torch.uint64}[x.dtype.itemsize]
        return torch.from_numpy(x.view(sig)).cuda().view(tdt)
    return torch.from_numpy(x).cuda()


def _keys(rng, dt, shape, dup=False):
    if np.dtype(dt).kind == "f":
        k = rng.standard_normal(shape).astype(dt)
        if dup:
            k = np.round(k * 4).astype(dt)
        return k
    info = np.iinfo(dt)
    k = rng.integers(info.min, info.max, size=shape, dtype=dt, endpoint=True)
    if dup:
        k %= 13
    return k


# 1025 / 4096: one CTA in shared memory; 65536 and 16385..40000: merge passes
@pytest.mark.parametrize("n", [1025, 4096, 16385, 65536])
@pytest.mark.parametrize("kdt", ["uint64", "int64", "uint32", "float32"])
@pytest.mark.parametrize("kind", ["merge", "rss"])
def test_big_rows_keys_only(n, kdt, kind, torch):
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(n)
    rows = 3 if n > 20000 else 9
    keys = _keys(rng, kdt, (rows, n), dup=True)
    keys[1] = _keys(rng, kdt, (n,))  # one row of (mostly) distinct keys
    for desc in (False, True):
        k, _ = batch.sort_rows(_t(torch, keys), kind=kind, descending=desc)
        exp = np.sort(keys, axis=1)
        if desc:
            exp = exp[:, ::-1]
        assert np.array_equal(k.cpu().numpy().view(keys.dtype), exp), (n, kdt, kind, desc)


@pytest.mark.parametrize("n", [1025, 4096, 65536])
def test_big_rows_vs_oracle(n, torch):
    """The oracle's reference RSS recursion on the same rows (no size cap)."""
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(7 + n)
    keys = _keys(rng, np.uint64, (2, n), dup=n != 65536)
    ek, _ = oracle.typed_sort_rows(keys, None, kind="rss")
    k, _ = batch.sort_rows(_t(torch, keys), kind="rss")
    assert np.array_equal(k.cpu().numpy(), ek)


@pytest.mark.parametrize("n", [1025, 9000, 20000])
@pytest.mark.parametrize("pdt", ["uint32", "uint64"])
def test_big_rows_unique_payload(n, pdt, torch):
    """(key, payload) lexicographic; 9000 / 20000 exceed the 12- and 16-byte
    item capacities (merge passes)."""
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(n + 3)
    keys = rng.integers(0, 50, size=(3, n)).astype(np.uint64)
    pay = rng.integers(0, 2**31, size=(3, n)).astype(pdt)
    for desc in (False, True):
        k, p = batch.sort_rows(_t(torch, keys), _t(torch, pay), kind="merge", descending=desc, tie="unique")
        kk, pp = k.cpu().numpy(), p.cpu().numpy().view(pay.dtype)
        for r in range(3):
            o = np.lexsort((pay[r], keys[r]))
            if desc:
                o = o[::-1]
            assert np.array_equal(kk[r], keys[r][o]) and np.array_equal(pp[r], pay[r][o]), (n, pdt, desc, r)
    if n == 1025:
        ek, ep = oracle.typed_sort_rows(keys, pay, unique=True, kind="rss")
        k, p = batch.sort_rows(_t(torch, keys), _t(torch, pay), kind="rss", tie="unique")
        assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy().view(pay.dtype), ep)


def test_big_rows_in_place(torch):
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(11)
    keys = _keys(rng, np.int64, (4, 40000))
    t = _t(torch, keys)
    batch.sort_rows(t, kind="merge", out_keys=t)
    assert np.array_equal(t.cpu().numpy(), np.sort(keys, axis=1))


def test_big_rows_ref_payload_rejected(torch):
    """REF-mode payload order (the reference's RSS replay) is not reproduced
    above 1024 items: the call refuses instead of returning another order."""
    from paper_2002_05599_b200 import batch
    from paper_2002_05599_b200.errors import ConfigurationError
    keys = np.zeros((2, 1025), dtype=np.uint64)
    with pytest.raises(ConfigurationError):
        batch.sort_rows(_t(torch, keys), _t(torch, keys), kind="rss", tie="ref")
