"""Generate the golden fixtures that pin the oracle and the CUDA path.

Run ONCE in the build container (the reference is NOT present on the GPU box):

    NETSORT_BACKEND=python PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It imports the reference package (`netsort`, pure-Python lane, which the
reference's own `test_backends.py` holds bit-identical to its compiled lane)
and records inputs/outputs of the hot-path entry points:

* networks.json   -- `networks.family_network(family, n)` comparator lists for
                     the 4 families x n=2..16 (reference networks.py:277-292),
                     the frozen BN size table (test_networks.py:11) and the
                     best sizes (test_networks.py:15-16);
* lcg.json        -- `lcg_next` / `fill_items` streams (netsort_core.c:38-50);
* fingerprint.json-- `fingerprint` (netsort_core.c:56-91) incl. the z-collision
                     path (test_backends.py:79-91);
* classify.npz    -- `classify_block_u64` for blocks 1..5 (netsort_core.c:270-300);
* net_rows.npz    -- `run_sorter_many(spec_network(fam, "4CmS"), rows)` for every
                     family and n=2..16 on 64-bit keys AND 2-bit duplicate-heavy
                     keys (the ties make the comparator DAG observable through
                     the ref payload, test_backends.py:162-177);
* rss_rows.npz    -- `run_sorter_many(spec_rss(cfg, base), rows)` for several
                     configs / bases / sizes, uniform and duplicate-heavy keys.

Only numbers are stored; no reference source is copied.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def main() -> None:
    if os.environ.get("NETSORT_BACKEND") != "python":
        print("set NETSORT_BACKEND=python (pure reference lane)", file=sys.stderr)
    from netsort import backend, networks as nw, registry
    from netsort.items import ITEM_DTYPE

    rng = np.random.default_rng(20020559)

    # ---- networks ---------------------------------------------------------
    nets = {}
    for fam in nw.FAMILY_KEYS:
        nets[fam] = {}
        for n in range(2, 17):
            net = nw.family_network(fam, n)
            nets[fam][str(n)] = [[c.low, c.high] for c in net.comparators]
    doc = {
        "source": "netsort.networks.family_network (reference networks.py:277-292)",
        "families": nets,
        "bn_sizes_0_20": [nw.generate_bose_nelson(n).size for n in range(21)],
        "best_depths": {str(n): nw.depth(nw.best_network(n)) for n in range(2, 17)},
        "bn_depths": {str(n): nw.depth(nw.generate_bose_nelson(n)) for n in range(2, 17)},
    }
    (OUT / "networks.json").write_text(json.dumps(doc, indent=0))

    # ---- LCG / fill -------------------------------------------------------
    s = 1
    stream = []
    for _ in range(64):
        s = backend.lcg_next(s)
        stream.append(s)
    fills = {}
    for seed in (1, 42, 0x5EED, 2147483646):
        arr = np.empty(37, dtype=ITEM_DTYPE)
        out = backend.fill_items(arr, seed)
        fills[str(seed)] = {"keys": arr["key"].tolist(), "refs": arr["ref"].tolist(),
                            "state_out": int(out)}
    (OUT / "lcg.json").write_text(json.dumps({"stream_from_1": stream, "fill": fills}))

    # ---- fingerprint ------------------------------------------------------
    fps = []
    for i in range(40):
        n = int(rng.integers(0, 40))
        keys = rng.integers(0, 2**64, size=n, dtype=np.uint64)
        if i % 5 == 0 and n > 2:
            keys[1] = 1  # z = 1 collides -> z bump path
        arr = np.zeros(n, dtype=ITEM_DTYPE)
        arr["key"] = keys
        v, z = backend.fingerprint(arr)
        fps.append({"keys": [int(k) for k in keys], "v": int(v), "z": int(z)})
    (OUT / "fingerprint.json").write_text(json.dumps(fps))

    # ---- classification ---------------------------------------------------
    cls = {}
    for block in range(1, 6):
        spl = np.sort(rng.integers(0, 2**64, size=3, dtype=np.uint64))
        keys = rng.integers(0, 2**64, size=257, dtype=np.uint64)
        keys[:3] = spl  # boundary keys (equal to a splitter) go low
        tags = backend.classify_block_u64(keys, int(spl[0]), int(spl[1]), int(spl[2]), block)
        cls[f"keys_{block}"] = keys
        cls[f"spl_{block}"] = spl
        cls[f"tags_{block}"] = np.asarray(tags, dtype=np.uint8)
    np.savez_compressed(OUT / "classify.npz", **cls)

    # ---- network rows -----------------------------------------------------
    net_rows = {}
    for fam in nw.FAMILY_KEYS:
        spec = registry.spec_network(fam, "4CmS")
        for n in range(2, 17):
            for kind, bits in (("u64", 64), ("dup", 2)):
                m = 48
                rows = np.empty((m, n), dtype=ITEM_DTYPE)
                if bits == 64:
                    rows["key"] = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
                else:
                    rows["key"] = rng.integers(0, 1 << bits, size=(m, n), dtype=np.uint64)
                rows["ref"] = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
                out = rows.copy()
                backend.run_sorter_many(spec, out)
                tag = f"{fam}_{n}_{kind}"
                net_rows[f"in_key_{tag}"] = rows["key"]
                net_rows[f"in_ref_{tag}"] = rows["ref"]
                net_rows[f"out_key_{tag}"] = out["key"]
                net_rows[f"out_ref_{tag}"] = out["ref"]
    np.savez_compressed(OUT / "net_rows.npz", **net_rows)

    # ---- RSS rows ---------------------------------------------------------
    rss_rows = {}
    cases = [
        ("332", "SN Best 4CmS"), ("333", "SN Best 4CmS"), ("341", "SN BN-L 4CmS"),
        ("315", "SN BN-R TCOp"), ("332", "IS Def"), ("391", "SN Best 4CmS"),
    ]
    meta = []
    for cfg, base in cases:
        spec = registry.spec_rss(cfg, base)
        for n in (17, 24, 32, 64, 100, 128, 256):
            for kind in ("u64", "dup", "sorted", "few"):
                m = 6 if n >= 128 else 10
                rows = np.empty((m, n), dtype=ITEM_DTYPE)
                if kind == "u64":
                    rows["key"] = rng.integers(0, 2**64, size=(m, n), dtype=np.uint64)
                elif kind == "dup":
                    rows["key"] = rng.integers(0, 4, size=(m, n), dtype=np.uint64)
                elif kind == "sorted":
                    rows["key"] = np.sort(rng.integers(0, 2**64, size=(m, n), dtype=np.uint64), axis=1)
                else:
                    vals = rng.integers(0, 2**64, size=16, dtype=np.uint64)
                    rows["key"] = vals[rng.integers(0, 16, size=(m, n))]
                rows["ref"] = np.arange(m * n, dtype=np.uint64).reshape(m, n)
                out = rows.copy()
                backend.run_sorter_many(spec, out)
                tag = f"{cfg}_{base.replace(' ', '-')}_{n}_{kind}"
                rss_rows[f"in_key_{tag}"] = rows["key"]
                rss_rows[f"out_key_{tag}"] = out["key"]
                rss_rows[f"out_ref_{tag}"] = out["ref"]
                meta.append({"tag": tag, "cfg": cfg, "base": base, "n": n, "kind": kind,
                             "spec": list(spec)})
    np.savez_compressed(OUT / "rss_rows.npz", **rss_rows)
    (OUT / "rss_meta.json").write_text(json.dumps(meta))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
