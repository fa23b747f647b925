"""GPU parity of Register Sample Sort (thread-per-array kernel for n <= 32,
warp-per-array kernel above) vs the oracle.

REF mode is bit-exact with the reference including payload order under key
ties, because the kernel replays the reference's LCG draws in depth-first
order (reference test_backends.py:145-177, test_acceptance.py A06/A07,
test_rss.py).
"""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
G = Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _items(keys, refs):
    a = np.empty(keys.shape, dtype=oracle.ITEM)
    a["key"], a["ref"] = keys, refs
    return a


def test_rss_matches_reference_golden(torch):
    from paper_2002_05599_b200 import backend, registry
    rss_rows = np.load(G / "rss_rows.npz")
    for meta in json.loads((G / "rss_meta.json").read_text()):
        t = meta["tag"]
        keys = rss_rows[f"in_key_{t}"]
        rows = _items(keys, np.arange(keys.size, dtype=np.uint64).reshape(keys.shape))
        spec = registry.spec_rss(meta["cfg"], meta["base"])
        assert list(spec) == meta["spec"]
        backend.run_sorter_many(spec, rows)
        assert np.array_equal(rows["key"], rss_rows[f"out_key_{t}"]), t
        assert np.array_equal(rows["ref"], rss_rows[f"out_ref_{t}"]), t


@pytest.mark.parametrize("cfg,base", [("332", "SN Best 4CmS"), ("333", "SN BN-L 4CmS"), ("341", "IS Def"),
                                      ("315", "SN BN-R TCOp"), ("391", "SN Best 4CmS"), ("311", "SN Best 4CmS")])
def test_rss_random_vs_oracle(cfg, base, torch):
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(int(cfg))
    spec = registry.spec_rss(cfg, base)
    fam = "best"
    kind_base = "ins" if base.startswith("IS") else "net"
    if base.startswith("SN"):
        fam = {"Best": "best", "BN-L": "bn-l", "BN-P": "bn-p", "BN-R": "bn-r"}[base.split()[1]]
    for n in (2, 16, 17, 20, 24, 31, 32, 33, 35, 64, 100, 255, 256, 257, 700, 1024):
        for gen in ("u64", "dup", "few", "sorted", "rev", "equal"):
            m = 64
            if gen == "u64":
                keys = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
            elif gen == "dup":
                keys = rng.integers(0, 4, size=(m, n), dtype=np.uint64)
            elif gen == "few":
                keys = rng.integers(0, 2**64, size=16, dtype=np.uint64)[rng.integers(0, 16, size=(m, n))]
            elif gen == "sorted":
                keys = np.sort(rng.integers(0, 2**64, size=(m, n), dtype=np.uint64), axis=1)
            elif gen == "rev":
                keys = np.sort(rng.integers(0, 2**64, size=(m, n), dtype=np.uint64), axis=1)[:, ::-1].copy()
            else:
                keys = np.full((m, n), 77, dtype=np.uint64)
            refs = np.arange(m * n, dtype=np.uint64).reshape(m, n)
            exp = _items(keys, refs)
            oracle.run_items(exp, kind="rss", family=fam, rss_cfg=cfg, base=kind_base)
            got = _items(keys, refs)
            backend.run_sorter_many(spec, got)
            assert np.array_equal(got, exp), (cfg, base, n, gen)


def test_rss_sort_api(torch):
    from paper_2002_05599_b200 import rss
    from paper_2002_05599_b200.items import items_from_keys, items_from_pairs
    arr = items_from_pairs([(42, i) for i in range(256)])
    rss.rss_sort(arr, rss.RssConfig.from_string("332"))
    assert arr["key"].tolist() == [42] * 256 and sorted(arr["ref"].tolist()) == list(range(256))
    arr = items_from_keys(list(range(300)))
    rss.rss_sort(arr, rss.RssConfig.from_string("341"))
    assert arr["key"].tolist() == list(range(300))
    rng = np.random.default_rng(12)
    cfg = rss.RssConfig.from_string("391")
    for n in range(17, 36):  # 16 < n < 4a: too small to sample
        keys = rng.integers(0, 2**64, size=n, dtype=np.uint64)
        arr = items_from_keys(keys)
        rss.rss_sort(arr, cfg)
        assert np.array_equal(arr["key"], np.sort(keys))


def test_insertion_kind_is_stable(torch):
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(3)
    for n in (2, 9, 16, 40, 300):
        keys = rng.integers(0, 3, size=(50, n), dtype=np.uint64)
        refs = np.arange(50 * n, dtype=np.uint64).reshape(50, n)
        got = _items(keys, refs)
        backend.run_sorter_many(registry.spec_insertion("Def"), got)
        order = np.argsort(keys, axis=1, kind="stable")
        assert np.array_equal(got["key"], np.take_along_axis(keys, order, 1))
        assert np.array_equal(got["ref"], np.take_along_axis(refs, order, 1))


@pytest.mark.parametrize("kdt", ["int64", "uint64", "uint32", "float32"])
@pytest.mark.parametrize("pdt", [None, "uint32", "uint64"])
def test_rss_typed_rows_vs_oracle(kdt, pdt, torch):
    from paper_2002_05599_b200 import batch
    rng = np.random.default_rng(7)
    for n in (32, 64, 128, 256, 300, 512):  # 257..512: the packed kernel's merge phase (keys-only / UNIQUE)
        for tie in (["unique"] if pdt is None else ["unique", "ref"]):
            for desc in (False, True):
                if kdt.startswith("float"):
                    keys = np.round(rng.standard_normal((300, n)) * 4).astype(kdt)
                else:
                    info = np.iinfo(kdt)
                    keys = rng.integers(info.min, info.max, size=(300, n), dtype=kdt, endpoint=True)
                    keys[::3] = keys[::3] % 5
                pay = None if pdt is None else rng.integers(0, 2**31, size=(300, n)).astype(pdt)
                ek, ep = oracle.typed_sort_rows(keys, pay, descending=desc, unique=tie == "unique", kind="rss")
                kt = torch.from_numpy(keys).cuda()
                pt = None
                if pay is not None:
                    pt = torch.from_numpy(pay.view(np.int32 if pdt == "uint32" else np.int64)).cuda()
                    pt = pt.view(torch.uint32 if pdt == "uint32" else torch.uint64)
                gk, gp = batch.sort_rows(kt, pt, kind="rss", descending=desc, tie=tie)
                assert np.array_equal(gk.cpu().numpy().view(np.uint8), ek.view(np.uint8)), (n, tie, desc)
                if pay is not None:
                    assert np.array_equal(gp.cpu().numpy().view(pay.dtype), ep), (n, tie, desc)


@pytest.mark.parametrize("n", [32, 64, 128, 256])
def test_cfg3_full_size_distributions(n, torch):
    """cfg3: 2^20 arrays of n int64 keys, four distributions; equal to torch.sort."""
    from paper_2002_05599_b200 import batch
    rows = 2**20
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(n)
    uni = torch.randint(-2**63, 2**63 - 1, (rows, n), dtype=torch.int64, device=dev, generator=gen)
    vals = torch.randint(-2**63, 2**63 - 1, (16,), dtype=torch.int64, device=dev, generator=gen)
    few = vals[torch.randint(0, 16, (rows, n), device=dev, generator=gen)]
    srt = torch.sort(uni, dim=1).values
    rev = torch.flip(srt, dims=[1]).contiguous()
    for name, x in (("uniform", uni), ("few16", few), ("sorted", srt), ("reverse", rev)):
        k, _ = batch.sort_rows(x, kind="rss")
        assert torch.equal(k, torch.sort(x, dim=1).values), name
    # a sampled subset against the oracle (full RSS replay)
    sub = uni[:512].cpu().numpy()
    ek, _ = oracle.typed_sort_rows(sub, None, kind="rss")
    k, _ = batch.sort_rows(uni[:512].contiguous(), kind="rss")
    assert np.array_equal(k.cpu().numpy(), ek)


@pytest.mark.parametrize("mode", ["ref_items", "unique_typed"])
def test_rss_thread_and_warp_kernels_agree(mode, torch, monkeypatch):
    """n <= 32 runs the thread-per-array kernel; NSG_RSS_WARP_ONLY=1 forces the
    warp kernel on the same rows: both must equal the oracle bit for bit."""
    from paper_2002_05599_b200 import backend, batch, registry
    rng = np.random.default_rng(99)
    spec = registry.spec_rss("332", "SN Best 4CmS")
    for n in (17, 23, 32):
        keys = rng.integers(0, 5, size=(301, n), dtype=np.uint64)
        refs = np.arange(keys.size, dtype=np.uint64).reshape(keys.shape)
        outs = []
        # (the packed sorter now serves REF rows of 17..256 items first;
        # NSG_RSS_FAITHFUL=1 keeps this test on the two draw-for-draw kernels)
        monkeypatch.setenv("NSG_RSS_FAITHFUL", "1")
        for warp_only in ("0", "1"):
            monkeypatch.setenv("NSG_RSS_WARP_ONLY", warp_only)
            if mode == "ref_items":
                got = _items(keys, refs)
                backend.run_sorter_many(spec, got)
                outs.append(got)
            else:
                k, p = batch.sort_rows(keys.astype(np.int64), refs.astype(np.uint32), kind="rss", tie="unique")
                outs.append((k, p))
        if mode == "ref_items":
            exp = _items(keys, refs)
            oracle.run_items(exp, kind="rss", family="best", rss_cfg="332", base="net")
            assert np.array_equal(outs[0], exp) and np.array_equal(outs[1], exp), n
        else:
            assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1]), n


@pytest.mark.parametrize("n", [20, 96, 256, 300, 512])
def test_ref_rows_fast_path_and_deferred_rows(n, torch, monkeypatch):
    """REF-mode items of 17..256 keys: rows with all-distinct keys are sorted by
    the packed sorter (their order is unique), rows with equal keys keep their
    input order there and are replayed draw for draw from a device list.  A
    batch mixing both, against the oracle, and against the draw-for-draw
    kernel alone (NSG_RSS_FAITHFUL=1)."""
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(1000 + n)
    m = 60_000
    keys = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
    dup = rng.random(m) < 0.05
    keys[dup, 1] = keys[dup, 0]                      # one equal pair
    heavy = rng.random(m) < 0.02
    keys[heavy] = keys[heavy] % np.uint64(3)         # duplicate-heavy rows
    keys[7] = np.sort(keys[7])
    refs = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
    spec = registry.spec_rss("332", "SN Best 4CmS")
    exp = _items(keys, refs)
    oracle.run_items(exp, kind="rss", family="best", rss_cfg="332", base="net")
    got = _items(keys, refs)
    backend.run_sorter_many(spec, got)
    assert np.array_equal(got, exp)
    dt = torch.from_numpy(_items(keys, refs).view(np.uint64).reshape(m, n, 2).view(np.int64)).cuda()
    backend.run_sorter_many(spec, dt)
    assert np.array_equal(dt.cpu().numpy().view(np.uint64).reshape(m, n * 2).view(oracle.ITEM), exp)
    monkeypatch.setenv("NSG_RSS_FAITHFUL", "1")
    slow = _items(keys, refs)
    backend.run_sorter_many(spec, slow)
    assert np.array_equal(slow, exp)


def test_ref_rows_deferred_list_overflow(torch):
    """More rows with equal keys than the deferred-row list holds (2^18): the
    draw-for-draw kernel then replays every row, from the output of the packed
    sorter (sorted rows and rows left in input order alike)."""
    from paper_2002_05599_b200 import backend, registry
    rng = np.random.default_rng(18)
    m, n = 300_000, 24
    keys = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
    keys[:, 5] = keys[:, 17]                         # every row has an equal pair
    keys[::7] %= np.uint64(4)
    keys[1::1000, 5] += np.uint64(1)                 # a few rows with distinct keys
    refs = np.arange(m * n, dtype=np.uint64).reshape(m, n)
    spec = registry.spec_rss("333", "SN BN-L 4CmS")
    exp = _items(keys, refs)
    oracle.run_items(exp, kind="rss", family="bn-l", rss_cfg="333", base="net", threads=8)
    got = _items(keys, refs)
    backend.run_sorter_many(spec, got)
    assert np.array_equal(got, exp)


def test_packed_sorters_lane_copy_fallback(torch, monkeypatch):
    """NSG_PK_NOBULK=1 takes the lane-copy staging of the packed sorters (what
    unaligned buffers get) through the padded-row and AoS layouts."""
    from paper_2002_05599_b200 import backend, batch, registry
    monkeypatch.setenv("NSG_PK_NOBULK", "1")
    rng = np.random.default_rng(44)
    for n in (32, 64, 100, 256):
        keys = rng.integers(-2**63, 2**63 - 1, size=(1501, n), dtype=np.int64)
        keys[::6] %= 4
        for kind in ("merge", "rss"):
            k, _ = batch.sort_rows(torch.from_numpy(keys).cuda(), kind=kind)
            assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1)), (kind, n)
        items = _items(keys.view(np.uint64), np.arange(keys.size, dtype=np.uint64).reshape(keys.shape))
        exp = items.copy()
        oracle.run_items(exp, kind="rss", rss_cfg="332")
        backend.run_sorter_many(registry.spec_rss("332"), items)
        assert np.array_equal(items, exp), n


@pytest.mark.parametrize("n", [2, 5, 11, 16])
def test_rss_rows_within_base_threshold(n, torch):
    """An RSS spec on rows of <= threshold items is its base case: the family's
    n-item network (C-ABI routes it to the network kernels).  Typed rows, REF
    and UNIQUE, and reference items with an insertion base (draw-for-draw kernel)."""
    from paper_2002_05599_b200 import backend, batch, registry
    rng = np.random.default_rng(70 + n)
    keys = rng.integers(0, 6, size=(3001, n)).astype(np.int64) - 3
    pay = rng.integers(0, 2**31, size=(3001, n)).astype(np.uint32)
    for tie in ("unique", "ref"):
        for desc in (False, True):
            ek, ep = oracle.typed_sort_rows(keys, pay, descending=desc, unique=tie == "unique", kind="rss")
            gk, gp = batch.sort_rows(torch.from_numpy(keys).cuda(),
                                     torch.from_numpy(pay.view(np.int32)).cuda().view(torch.uint32),
                                     kind="rss", descending=desc, tie=tie)
            assert np.array_equal(gk.cpu().numpy(), ek), (tie, desc)
            assert np.array_equal(gp.cpu().numpy().view(np.uint32), ep), (tie, desc)
    for cfg, base, fam, kb in (("332", "SN BN-L 4CmS", "bn-l", "net"), ("341", "IS Def", "best", "ins")):
        items = _items(keys.view(np.uint64), np.arange(keys.size, dtype=np.uint64).reshape(keys.shape))
        exp = items.copy()
        oracle.run_items(exp, kind="rss", family=fam, rss_cfg=cfg, base=kb)
        backend.run_sorter_many(registry.spec_rss(cfg, base), items)
        assert np.array_equal(items, exp), (cfg, base)
