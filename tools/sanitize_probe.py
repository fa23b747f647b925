"""Small launches of every device sorter, each checked against numpy / the
oracle -- run against the CHECKED build (device-side bounds and invariant
checks, NSG_DCHECK in csrc/common.cuh; compute-sanitizer is closed on this
GPU pool):

    python tools/sanitize_probe.py --build-checked       # here: variants/checked/libnsg.so
    NSG_LIB_PATH=variants/checked/libnsg.so python tools/sanitize_probe.py   # on the GPU

Shapes are tiny (a few hundred rows) so the instrumented run stays short, but
they cover the odd paths: non-power-of-two rows, the tail group of a staging
ring, payloads, descending floats, CSR segments of every length class, and
rows above 1024 items (tile sort + merge passes).
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2002_05599_b200 import backend, batch, registry
    import oracle

    rng = np.random.default_rng(5)
    dev = torch.device("cuda")

    def t(x):
        x = np.ascontiguousarray(x)
        if x.dtype == np.uint64:
            return torch.from_numpy(x.view(np.int64)).to(dev).view(torch.uint64)
        if x.dtype == np.uint32:
            return torch.from_numpy(x.view(np.int32)).to(dev).view(torch.uint32)
        return torch.from_numpy(x).to(dev)

    checks = 0
    # network kernels (n <= 16), keys-only and key + u32 payload (UNIQUE)
    for n in (3, 8, 13, 16):
        keys = rng.integers(0, 2**64, size=(333, n), dtype=np.uint64)
        pay = rng.integers(0, 2**32, size=(333, n), dtype=np.uint64).astype(np.uint32)
        k, _ = batch.sort_rows(t(keys))
        assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1))
        k, p = batch.sort_rows(t(keys), t(pay), tie="unique")
        ek, ep = oracle.typed_sort_rows(keys, pay, unique=True)
        assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy(), ep)
        checks += 2
    # AoS reference items, REF mode
    items = np.empty((200, 11), dtype=oracle.ITEM)
    items["key"] = rng.integers(0, 3, size=(200, 11), dtype=np.uint64)
    items["ref"] = np.arange(2200, dtype=np.uint64).reshape(200, 11)
    exp = items.copy()
    oracle.run_items(exp, kind="network", family="bn-l")
    backend.run_sorter_many(registry.spec_network("bn-l", "4CmS"), items)
    assert np.array_equal(items, exp)
    checks += 1
    # packed-key warp sorters (merge, rss) and the faithful RSS / warp merge
    for n in (17, 64, 100, 256, 300, 1000):
        keys = rng.integers(-2**63, 2**63 - 1, size=(77, n), dtype=np.int64)
        keys[::4] %= 5
        for kind in ("merge", "rss"):
            k, _ = batch.sort_rows(t(keys), kind=kind)
            assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1)), (kind, n)
            checks += 1
        pay = rng.integers(0, 2**32, size=(77, n), dtype=np.uint64)
        k, p = batch.sort_rows(t(keys), t(pay), kind="rss", tie="ref")
        ek, ep = oracle.typed_sort_rows(keys, pay, unique=False, kind="rss")
        assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy(), ep), n
        checks += 1
    # floats descending (order transform paths)
    keys = np.round(rng.standard_normal((55, 40)) * 3).astype(np.float32)
    k, _ = batch.sort_rows(t(keys), kind="merge", descending=True)
    assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1)[:, ::-1])
    checks += 1
    # rows above 1024 items: CTA shared-memory sort and merge passes
    for n in (1500, 20000):
        keys = rng.integers(0, 2**64, size=(2, n), dtype=np.uint64)
        k, _ = batch.sort_rows(t(keys), kind="merge")
        assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1)), n
        checks += 1
    # CSR segments: every length class, long (warp RSS) and above 1024 (CTA)
    lengths = np.concatenate([oracle.geometric_lengths(3000, seed=9),
                              np.array([0, 17, 300, 1024, 1025, 2000], dtype=np.uint32)])
    off = np.zeros(len(lengths) + 1, dtype=np.uint32)
    np.cumsum(lengths, out=off[1:])
    w = rng.random(int(off[-1])).astype(np.float32)
    ids = rng.integers(0, 2**26, size=int(off[-1])).astype(np.uint32)
    gk, gp = batch.sort_segments(t(off), t(w), t(ids), descending=True, tie="unique")
    ek, ep = oracle.typed_sort_segments(off, w, ids, descending=True, unique=True)
    assert np.array_equal(gk.cpu().numpy(), ek) and np.array_equal(gp.cpu().numpy(), ep)
    checks += 1
    # padded row staging of the packed sorters (full power-of-two rows, >= 4
    # rows per group) including a ragged last group, with and without a payload
    for n in (32, 64, 128):
        keys = rng.integers(-2**63, 2**63 - 1, size=(1003, n), dtype=np.int64)
        keys[::5] %= 3
        pay = rng.integers(0, 2**63, size=(1003, n), dtype=np.uint64)
        for kind in ("merge", "rss"):
            k, _ = batch.sort_rows(t(keys), kind=kind)
            assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1)), (kind, n)
            k, p = batch.sort_rows(t(keys), t(pay), kind=kind, tie="unique")
            ek, ep = oracle.typed_sort_rows(keys, pay, unique=True, kind="rss")
            assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy(), ep), (kind, n)
            checks += 2
    # CSR software pipeline: more tiles than CTAs (every CTA walks several
    # tiles) with stretches of oversized tiles (synchronous sub-tiles) between
    lengths = oracle.geometric_lengths(900_000, seed=11).astype(np.uint32)
    for lo in range(50_000, 850_000, 90_000):
        lengths[lo:lo + 3000] = 16
    off = np.zeros(len(lengths) + 1, dtype=np.uint32)
    np.cumsum(lengths, out=off[1:])
    w = (rng.integers(-30, 30, int(off[-1])) / 4.0).astype(np.float32)
    ids = rng.integers(0, 2**26, size=int(off[-1])).astype(np.uint32)
    for tie in ("unique", "ref"):
        gk, gp = batch.sort_segments(t(off), t(w), t(ids), descending=True, tie=tie)
        ek, ep = oracle.typed_sort_segments(off, w, ids, descending=True, unique=tie == "unique")
        assert np.array_equal(gk.cpu().numpy().view(np.uint32), ek.view(np.uint32))
        assert np.array_equal(gp.cpu().numpy(), ep)
        checks += 1
    # midsort (513..10240 items: packed chunks + merge-path passes), ragged tails,
    # and the robust second packing (small keys of both signs)
    for n in (513, 1000, 1024, 3000, 10240):
        keys = rng.integers(-2**63, 2**63 - 1, size=(37, n), dtype=np.int64)
        keys[::3] = rng.integers(-500, 500, size=keys[::3].shape)
        pay = rng.integers(0, 2**32, size=(37, n), dtype=np.uint64).astype(np.uint32)
        for kind in ("merge", "rss"):
            k, _ = batch.sort_rows(t(keys), kind=kind)
            assert np.array_equal(k.cpu().numpy(), np.sort(keys, axis=1)), (kind, n)
            checks += 1
        if n <= 6000:
            k, p = batch.sort_rows(t(keys), t(pay), kind="merge", tie="unique")
            ek, ep = oracle.typed_sort_rows(keys, pay, unique=True, kind="rss")
            assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy().view(np.uint32), ep), n
            checks += 1
    # REF items through the packed kernel + deferred rows (AoS staging)
    for n in (40, 256, 400):
        items = np.empty((500, n), dtype=oracle.ITEM)
        items["key"] = rng.integers(0, 2**64, size=(500, n), dtype=np.uint64)
        items["key"][::5] %= np.uint64(4)
        items["ref"] = np.arange(500 * n, dtype=np.uint64).reshape(500, n)
        exp = items.copy()
        oracle.run_items(exp, kind="rss", rss_cfg="332")
        backend.run_sorter_many(registry.spec_rss("332"), items)
        assert np.array_equal(items, exp), n
        checks += 1
    torch.cuda.synchronize()
    print(f"sanitize probe ok ({checks} checks)")


if __name__ == "__main__":
    if "--build-checked" in sys.argv:
        from paper_2002_05599_b200.build import build
        d = Path(__file__).resolve().parent.parent / "variants" / "checked"
        print(build(defines=("NSG_CHECKED=1",), lib_path=d / "libnsg.so", obj_dir=d / "obj", jobs=8))
    else:
        main()
