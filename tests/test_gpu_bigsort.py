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


def _items(keys, refs):
    it = np.empty(keys.shape, dtype=oracle.ITEM)
    it["key"] = keys
    it["ref"] = refs
    return it


@pytest.mark.parametrize("cfg,base", [("332", "SN Best 4CmS"), ("315", "SN BN-R TCOp"), ("391", "IS Def")])
@pytest.mark.parametrize("n", [1025, 4096, 30000])
def test_big_rows_ref_mode_rss_vs_oracle(cfg, base, n, torch):
    """The reference's tie order above 1024 items (csrc/rssbig.cu): AoS items
    through run_sorter_many, duplicate-heavy keys so the payload order under
    ties shows every draw, bucket and base case."""
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(n + int(cfg))
    spec = registry.spec_rss(cfg, base)
    fam = "best" if "Best" in base or base.startswith("IS") else "bn-r"
    kind_base = "ins" if base.startswith("IS") else "net"
    m = 3
    keys = rng.integers(0, 40, size=(m, n), dtype=np.uint64)
    keys[1] = rng.integers(0, 2**64, size=n, dtype=np.uint64)  # distinct
    keys[2, : n // 2] = 7                                     # one huge run of ties
    refs = np.arange(m * n, dtype=np.uint64).reshape(m, n)
    exp = _items(keys, refs)
    oracle.run_items(exp, kind="rss", family=fam, rss_cfg=cfg, base=kind_base)
    got = _items(keys, refs)
    backend.run_sorter_many(spec, got)
    assert np.array_equal(got, exp), (cfg, base, n)


def test_big_rows_rss_sort_and_typed_ref(torch):
    """rss.rss_sort (the reference's API, no size cap) and typed REF-mode rows
    with a payload above 1024 items equal the oracle."""
    from paper_2002_05599_b200 import batch, rss
    from paper_2002_05599_b200.items import items_from_pairs
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 9, size=3000, dtype=np.uint64)
    arr = items_from_pairs(zip(keys.tolist(), range(3000)))
    rss.rss_sort(arr, rss.RssConfig.from_string("332"))
    exp = _items(keys.reshape(1, -1), np.arange(3000, dtype=np.uint64).reshape(1, -1))
    oracle.run_items(exp, kind="rss", family="best", rss_cfg="332")
    assert np.array_equal(arr, exp[0])
    for kdt in ("int64", "uint32", "float32"):
        k = rng.integers(-5, 5, size=(2, 2500)).astype(kdt)
        pay = rng.integers(0, 2**31, size=(2, 2500)).astype(np.uint32)
        for desc in (False, True):
            ek, ep = oracle.typed_sort_rows(k, pay, descending=desc, unique=False, kind="rss")
            gk, gp = batch.sort_rows(_t(torch, k), _t(torch, pay), kind="rss", tie="ref", descending=desc)
            assert np.array_equal(gk.cpu().numpy().view(k.dtype), ek) and np.array_equal(gp.cpu().numpy(), ep), \
                (kdt, desc)


def test_big_rows_insertion_kind_is_stable(torch):
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 6, size=(2, 2000), dtype=np.uint64)
    refs = np.arange(4000, dtype=np.uint64).reshape(2, 2000)
    got = _items(keys, refs)
    backend.run_sorter_many(registry.spec_insertion("Def"), got)
    for r in range(2):
        o = np.argsort(keys[r], kind="stable")
        assert np.array_equal(got[r]["key"], keys[r][o]) and np.array_equal(got[r]["ref"], refs[r][o])
