"""GPU parity of the merge sorter (n > 16: odd-even merge networks at 32/64,
warp bitonic merge up to 1024) vs the oracle / numpy.  Keys-only and UNIQUE
(key, payload) outputs are unique, so they must equal np.sort / np.lexsort
and the reference-restating oracle bit for bit."""

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


@pytest.mark.parametrize("n", [17, 31, 32, 33, 64, 65, 100, 128, 200, 256, 257, 512, 1000, 1024])
@pytest.mark.parametrize("kdt", ["uint64", "int64", "uint32", "float32"])
def test_merge_keys_only(n, kdt, torch):
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(n)
    rows = 777
    if kdt.startswith("float"):
        keys = np.round(rng.standard_normal((rows, n)) * 8).astype(kdt)
    else:
        info = np.iinfo(kdt)
        keys = rng.integers(info.min, info.max, size=(rows, n), dtype=kdt, endpoint=True)
        keys[::2] %= 7
    for desc in (False, True):
        k, _ = batch.sort_rows(_t(torch, keys), kind="merge", descending=desc)
        exp = np.sort(keys, axis=1)
        if desc:
            exp = exp[:, ::-1]
        assert np.array_equal(k.cpu().numpy().view(keys.dtype), exp), (n, kdt, desc)


@pytest.mark.parametrize("n", [20, 32, 64, 96, 128, 256, 300, 512, 700])
@pytest.mark.parametrize("pdt", ["uint32", "uint64"])
def test_merge_unique_payload_vs_oracle(n, pdt, torch):
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(n + 1)
    keys = rng.integers(0, 9, size=(500, n)).astype(np.uint64)
    pay = rng.integers(0, 2**31, size=(500, n)).astype(pdt)
    for desc in (False, True):
        ek, ep = oracle.typed_sort_rows(keys, pay, descending=desc, unique=True, kind="rss")
        k, p = batch.sort_rows(_t(torch, keys), _t(torch, pay), kind="merge", descending=desc, tie="unique")
        assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy().view(pay.dtype), ep)


def test_merge_rejects_ref_mode_payload(torch):
    from paper_2002_05599_b200 import batch
    from paper_2002_05599_b200.errors import ConfigurationError
    keys = np.zeros((4, 40), dtype=np.uint64)
    with pytest.raises(ConfigurationError):
        batch.sort_rows(_t(torch, keys), _t(torch, keys), kind="merge", tie="ref")


@pytest.mark.parametrize("n", [32, 64, 128, 256])
def test_cfg3_merge_full_size(n, torch):
    from paper_2002_05599_b200 import batch
    rows = 2**20
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(n)
    uni = torch.randint(-2**63, 2**63 - 1, (rows, n), dtype=torch.int64, device=dev, generator=g)
    vals = torch.randint(-2**63, 2**63 - 1, (16,), dtype=torch.int64, device=dev, generator=g)
    few = vals[torch.randint(0, 16, (rows, n), device=dev, generator=g)]
    srt = torch.sort(uni, dim=1).values
    rev = torch.flip(srt, dims=[1]).contiguous()
    for name, x in (("uniform", uni), ("few16", few), ("sorted", srt), ("reverse", rev)):
        k, _ = batch.sort_rows(x, kind="merge")
        assert torch.equal(k, torch.sort(x, dim=1).values), name


@pytest.mark.parametrize("n", [64, 128, 256, 512])
@pytest.mark.parametrize("kdt", ["uint64", "int64", "uint32"])
def test_merge_path_sentinel_ties(n, kdt, torch):
    """Rows full of the largest key (the merge path's +inf sentinel value in
    the ordered space -- all ones; INT64_MAX for signed keys ascending, the
    minimum for descending) merge to the same values as np.sort: a lane whose
    A run is exhausted may emit the sentinel for an equal B item."""
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(n + 7)
    info = np.iinfo(kdt)
    rows = 999
    choices = np.array([info.max, info.max - 1, info.min, 0, 5], dtype=kdt)
    keys = choices[rng.integers(0, 5, size=(rows, n))]
    keys[::3] = info.max
    keys[1::3, : n // 2] = info.min
    for desc in (False, True):
        k, _ = batch.sort_rows(_t(torch, keys), kind="merge", descending=desc)
        exp = np.sort(keys, axis=1)
        if desc:
            exp = exp[:, ::-1]
        assert np.array_equal(k.cpu().numpy().view(keys.dtype), exp), (n, kdt, desc)
    if kdt == "uint64":  # UNIQUE (key, payload) with all-ones payloads as well
        pay = np.where(rng.integers(0, 2, size=(rows, n)) == 1, np.uint64(2**64 - 1), np.uint64(3))
        for desc in (False, True):
            ek, ep = oracle.typed_sort_rows(keys, pay, descending=desc, unique=True, kind="rss")
            k, p = batch.sort_rows(_t(torch, keys), _t(torch, pay), kind="merge", descending=desc, tie="unique")
            assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy(), ep), (n, desc)


@pytest.mark.parametrize("n", [32, 100, 256, 512])
@pytest.mark.parametrize("kind", ["merge", "rss"])
def test_sign_extended_small_keys(n, kind, torch):
    """int64 keys of small magnitude and both signs: in the ordered space they
    straddle 2^63, so the common-prefix window of the packed words sees the
    sign only.  The merge phase packs the group a second time (distance to the
    row minimum), the RSS phase re-sorts the rows exactly: same output."""
    from paper_2002_05599_b200 import batch
    from paper_2002_05599_b200._lib import lib
    rng = np.random.default_rng(n)
    keys = rng.integers(-1000, 1000, size=(4000, n), dtype=np.int64)
    keys[::9] = rng.integers(-2**40, 2**40, size=keys[::9].shape, dtype=np.int64)
    pay = rng.integers(0, 2**32, size=keys.shape, dtype=np.uint64).astype(np.uint32)
    k, _ = batch.sort_rows(_t(torch, keys), kind=kind)
    assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1))
    ek, ep = oracle.typed_sort_rows(keys, pay, unique=True, kind="rss")
    k, p = batch.sort_rows(_t(torch, keys), _t(torch, pay), kind=kind, tie="unique")
    assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy().view(np.uint32), ep)
