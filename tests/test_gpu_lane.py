"""Device lane utilities vs the reference's goldens and the oracle
(SURVEY 8(f) items 1-2): ns_fill, ns_fp_at/ns_fp_search, ns_scan_sorted,
ns_measure_air -- here computed by libnsg.so on the GPU."""

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


def _items(pairs):
    a = np.zeros(len(pairs), dtype=oracle.ITEM)
    if pairs:
        a["key"] = np.array([k for k, _ in pairs], dtype=np.uint64)
        a["ref"] = np.array([r for _, r in pairs], dtype=np.uint64)
    return a


def test_fill_items_matches_golden(torch):
    from paper_2002_05599_b200 import backend
    lcg = json.loads((G / "lcg.json").read_text())
    for seed, rec in lcg["fill"].items():
        a = np.empty(37, dtype=oracle.ITEM)
        st = backend.fill_items(a, int(seed))
        assert a["key"].tolist() == rec["keys"] and a["ref"].tolist() == rec["refs"]
        assert st == rec["state_out"]


@pytest.mark.parametrize("seed", [1, 42, 0x5EED, 2147483646, 2147483647, 0xFFFFFFFF, 0])
def test_fill_items_vs_oracle(seed, torch):
    # test_backends.py:64-71 (native == pure for seeds 1, 42, 2^31-2), plus
    # out-of-range states the u32 argument admits
    from paper_2002_05599_b200 import backend
    a, b = np.empty(97, dtype=oracle.ITEM), np.empty(97, dtype=oracle.ITEM)
    assert backend.fill_items(a, seed) == oracle.fill_items(b, seed)
    assert np.array_equal(a, b)


def test_fill_items_jump_ahead_large(torch):
    """1,000,003 items: every thread jumps ahead to its run; spot-check against
    the closed form seed * 48271^k mod (2^31-1) and the sequential oracle."""
    from paper_2002_05599_b200 import backend
    n, seed = 1_000_003, 12345
    t = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    st = backend.fill_items(t, seed)
    assert st == oracle.lcg_jump(seed, 2 * n)
    h = t.cpu().numpy().view(np.uint64)
    rng = np.random.default_rng(3)
    for i in list(rng.integers(0, n, 500)) + [0, 1, 7, 8, 9, n - 1]:
        assert int(h[i, 0]) == oracle.lcg_jump(seed, 2 * int(i) + 1)
        assert int(h[i, 1]) == oracle.lcg_jump(seed, 2 * int(i) + 2)
    b = np.empty(4099, dtype=oracle.ITEM)
    oracle.fill_items(b, seed)
    assert np.array_equal(h[:4099, 0], b["key"]) and np.array_equal(h[:4099, 1], b["ref"])


def test_fill_items_empty(torch):
    from paper_2002_05599_b200 import backend
    assert backend.fill_items(np.empty(0, dtype=oracle.ITEM), 77) == 77


def test_fingerprint_matches_golden(torch):
    from paper_2002_05599_b200 import backend
    for rec in json.loads((G / "fingerprint.json").read_text()):
        a = _items([(k, 0) for k in rec["keys"]])
        assert backend.fingerprint(a) == (rec["v"], rec["z"])


def test_fingerprint_z_collision_path(torch):
    # test_backends.py:80-91
    from paper_2002_05599_b200 import backend
    p = backend.FP_PRIME
    assert backend.fingerprint(_items([(1, 0), (5, 0)]), z=1) == oracle.fingerprint([1, 5], z=1)
    assert backend.fingerprint(_items([(1, 0), (5, 0)]), z=1)[1] == 2
    assert backend.fingerprint(_items([(p + 3, 0)]), z=3) == oracle.fingerprint([p + 3], z=3)
    assert backend.fingerprint(_items([])) == (1, 1)


def test_fingerprint_large_and_permutation_invariant(torch):
    """A 200,003-item array: the device tree product equals the sequential
    oracle and is invariant under a permutation (test_acceptance.py:243-265)."""
    from paper_2002_05599_b200 import backend
    rng = np.random.default_rng(10)
    n = 200_003
    keys = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    a = _items(list(zip(keys.tolist(), [0] * n)))
    v = backend.fingerprint(a)
    assert v == oracle.fingerprint(keys.tolist())
    assert backend.fingerprint(a[rng.permutation(n)].copy()) == v
    m = a.copy()
    m["key"][12345] += np.uint64(1)
    assert backend.fingerprint(m, z=v[1]) != v


def test_fingerprint_rows_vs_oracle(torch):
    from paper_2002_05599_b200 import _lib
    l = _lib.lib()
    rng = np.random.default_rng(5)
    rows, n = 3001, 13
    keys = rng.integers(0, 2**64, size=rows * n, dtype=np.uint64)
    for kb, col in ((8, keys), (4, (keys >> np.uint64(40)).astype(np.uint32))):
        t = torch.from_numpy(col.view(np.int64 if kb == 8 else np.int32)).cuda()
        out = torch.empty(rows, dtype=torch.int64, device="cuda")
        _lib.check(l.nsg_fingerprint_rows(t.data_ptr(), kb, kb, rows, n, 7, out.data_ptr(),
                                          _lib.current_stream_handle()))
        got = out.cpu().numpy().view(np.uint64)
        for r in range(0, rows, 97):
            want = 1
            for k in col[r * n:(r + 1) * n].tolist():
                want = want * ((7 - int(k) % oracle.FP_PRIME) % oracle.FP_PRIME) % oracle.FP_PRIME
            assert int(got[r]) == want


def test_check_sorted_cases(torch):
    # test_backends.py:94-100
    import random
    from paper_2002_05599_b200 import backend
    rng = random.Random(31)
    cases = [[], [1], [1, 1, 2], [2, 1], list(range(50))]
    cases += [[rng.getrandbits(8) for _ in range(20)] for _ in range(20)]
    cases += [[2**64 - 1, 0], [0, 2**63, 2**64 - 1]]
    for keys in cases:
        arr = _items([(k, 0) for k in keys])
        assert backend.check_sorted(arr) == all(a <= b for a, b in zip(keys, keys[1:]))
    big = np.sort(np.random.default_rng(1).integers(0, 2**64, 1 << 20, dtype=np.uint64))
    t = torch.from_numpy(np.stack([big, big], 1).view(np.int64)).cuda()
    assert backend.check_sorted(t)
    t[777_777, 0] = 0
    assert not backend.check_sorted(t)


@pytest.mark.parametrize("kind,size", [("network", 8), ("network", 16), ("network", 1), ("rss", 64)])
def test_measure_array_in_row(kind, size, torch):
    from paper_2002_05599_b200 import backend, registry
    spec = registry.spec_network("best", "4CmS") if kind == "network" else registry.spec_rss("332")
    ns = backend.measure_array_in_row(spec, size, 1 << 14, 4242)
    assert isinstance(ns, int) and ns > 0


def test_measure_array_in_row_rejects_network_size(torch):
    from paper_2002_05599_b200 import backend, registry
    from paper_2002_05599_b200.errors import UnsupportedSize
    with pytest.raises(UnsupportedSize):
        backend.measure_array_in_row(registry.spec_network("best", "4CmS"), 17, 100, 1)


def test_array_in_row_records(torch):
    """The reference's ArrayInRow loop (bench.py:148-185) over the device lane:
    records carry nanoseconds per subarray and round-trip through CSV."""
    import io
    from paper_2002_05599_b200 import measure
    recs = measure.array_in_row("SN Best 4CmS", 8, 1 << 20, 3, measure.SeedSequence(7),
                                cache_bytes=126 * 2**20)
    assert [r.measure_index for r in recs] == [0, 1, 2]
    assert all(r.timer_kind == "nanos" and r.sorter == "SN Best 4CmS" and 0 < r.cost < 1e3 for r in recs)
    assert measure.read_records(io.StringIO(measure.records_to_csv_text(recs))) == recs
