"""API edge cases and error behaviour on the device lane (mirrors the
reference's contracts: empty / single-item inputs are no-ops, out-of-range
sizes raise UnsupportedSize, rejected specs raise ConfigurationError)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def test_empty_and_trivial_shapes(torch):
    from paper_2002_05599_b200 import backend, batch, registry
    from paper_2002_05599_b200.items import ITEM_DTYPE
    spec = registry.spec_network("best", "4CmS")
    for m, n in ((0, 8), (5, 0), (0, 0)):
        rows = np.zeros((m, n), dtype=ITEM_DTYPE)
        backend.run_sorter_many(spec, rows)          # no-op, no error
    rows = np.zeros((4, 1), dtype=ITEM_DTYPE)
    rows["key"] = [[3], [1], [2], [0]]
    backend.run_sorter_many(spec, rows)              # n < 2: untouched (ns_run_sorter)
    assert rows["key"].ravel().tolist() == [3, 1, 2, 0]
    k = np.array([[5], [4]], dtype=np.uint32)
    out, _ = batch.sort_rows(k)                      # n = 1: identity copy
    assert np.array_equal(out, k)
    z = torch.empty((0, 7), dtype=torch.int64, device="cuda")
    zo, _ = batch.sort_rows(z)
    assert zo.shape == (0, 7)


def test_error_mapping(torch):
    from paper_2002_05599_b200 import backend, batch, registry, smallsort
    from paper_2002_05599_b200.errors import ConfigurationError, UnsupportedSize
    from paper_2002_05599_b200.items import ITEM_DTYPE, items_from_keys
    rows = np.zeros((3, 17), dtype=ITEM_DTYPE)
    with pytest.raises(UnsupportedSize):
        backend.run_sorter_many(registry.spec_network("bn-l", "ISwp"), rows)
    with pytest.raises(ConfigurationError):
        backend.run_sorter_many(registry.spec_hybrid("SN Best 4CmS"), np.zeros((3, 8), dtype=ITEM_DTYPE))
    with pytest.raises(ConfigurationError):
        backend.run_sorter_many(registry.spec_network("best", "4CmS"), np.zeros(8, dtype=ITEM_DTYPE))
    with pytest.raises(ConfigurationError):  # not C-contiguous
        backend.run_sorter_many(registry.spec_network("best", "4CmS"),
                                np.zeros((8, 8), dtype=ITEM_DTYPE)[:, ::2])
    with pytest.raises(UnsupportedSize):
        batch.sort_rows(np.zeros((2, 17), dtype=np.uint64))
    with pytest.raises(UnsupportedSize):
        smallsort.sort_small(items_from_keys(range(20)), 17, "SN Best 4CmS")
    with pytest.raises(UnsupportedSize):
        smallsort.sort_small(items_from_keys([3, 2, 1]), 3, "RSS 332 IS Def")
    # RSS above 1024 items (no size cap, as the reference): keys-only through the CTA sorter
    k, _ = batch.sort_rows(np.arange(2200, dtype=np.uint64)[::-1].reshape(2, 1100).copy(), kind="rss")
    assert np.array_equal(k, np.sort(np.arange(2200, dtype=np.uint64)[::-1].reshape(2, 1100), axis=1))


def test_sort_small_dispatch_and_insertion(torch):
    from paper_2002_05599_b200 import smallsort
    from paper_2002_05599_b200.items import items_from_pairs
    rng = np.random.default_rng(777)
    for _ in range(20):
        keys = rng.integers(0, 4, size=8)
        a = items_from_pairs(zip(keys, range(8)))
        b = a.copy()
        smallsort.sort_small(a, 8, "SN Best 4CmS")
        smallsort.insertion_sort(b, 8, "Def")
        assert np.array_equal(a["key"], b["key"])
        order = np.argsort(keys, kind="stable")      # insertion sort is stable by key
        assert b["ref"].tolist() == order.tolist()
    big = items_from_pairs(zip(rng.integers(0, 9, size=300), range(300)))
    smallsort.sort_small(big, 300, "IS Def")
    assert np.all(np.diff(big["key"].astype(np.int64)) >= 0)


def test_rss_host_and_device_paths_agree(torch):
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(9)
    rows = np.empty((300, 100), dtype=oracle.ITEM)
    rows["key"] = rng.integers(0, 5, size=(300, 100), dtype=np.uint64)
    rows["ref"] = np.arange(30000, dtype=np.uint64).reshape(300, 100)
    dev = torch.from_numpy(rows.view(np.uint64).reshape(300, 100, 2).astype(np.int64)).cuda()
    spec = registry.spec_rss("332")
    host = rows.copy()
    backend.run_sorter_many(spec, host)
    backend.run_sorter_many(spec, dev)
    got = dev.cpu().numpy().view(np.uint64)
    assert np.array_equal(got[:, :, 0], host["key"]) and np.array_equal(got[:, :, 1], host["ref"])
    exp = rows.copy()
    oracle.run_items(exp, kind="rss", rss_cfg="332")
    assert np.array_equal(host, exp)


def test_stream_ordering_on_side_stream(torch):
    from paper_2002_05599_b200 import batch
    s = torch.cuda.Stream()
    x = torch.randint(-2**63, 2**63 - 1, (1 << 16, 12), dtype=torch.int64, device="cuda")
    with torch.cuda.stream(s):
        y, _ = batch.sort_rows(x)
    s.synchronize()
    assert torch.equal(y, torch.sort(x, dim=1).values)
