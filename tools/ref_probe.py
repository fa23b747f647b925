"""Time the reference-shaped RSS entry (run_sorter_many on AoS (key, ref)
items, REF mode) and typed REF rows on the device, distinct and duplicate-heavy
keys, against the draw-for-draw kernel alone (NSG_RSS_FAITHFUL=1):

    python tools/ref_probe.py [--ns 32,64,128,256] [--rows 1048576]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="32,64,128,256")
    ap.add_argument("--rows", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import oracle
    from paper_2002_05599_b200 import backend, registry
    dev = torch.device("cuda")
    spec = registry.spec_rss("332")
    for n in [int(x) for x in a.ns.split(",")]:
        g = torch.Generator(device=dev).manual_seed(n)
        for dist in ("distinct", "dup1pct", "few16"):
            keys = torch.randint(-2**63, 2**63 - 1, (a.rows, n), dtype=torch.int64, device=dev, generator=g)
            if dist == "few16":
                vals = torch.randint(-2**63, 2**63 - 1, (a.rows, 16), dtype=torch.int64, device=dev, generator=g)
                keys = torch.gather(vals, 1, torch.randint(0, 16, (a.rows, n), device=dev, generator=g))
            elif dist == "dup1pct":  # one row in a hundred carries a duplicated key
                keys[::100, 1] = keys[::100, 0]
            items = torch.empty((a.rows, n, 2), dtype=torch.int64, device=dev)
            items[:, :, 0] = keys
            items[:, :, 1] = torch.arange(a.rows * n, device=dev).view(a.rows, n)
            work = torch.empty_like(items)
            # parity of a prefix against the oracle (reference restatement)
            work.copy_(items)
            backend.run_sorter_many(spec, work)
            sub = items[:256].cpu().numpy().view(np.uint64)
            exp = np.empty((256, n), dtype=oracle.ITEM)
            exp["key"], exp["ref"] = sub[:, :, 0], sub[:, :, 1]
            oracle.run_items(exp, kind="rss", rss_cfg="332")
            got = work[:256].cpu().numpy().view(np.uint64)
            ok = bool(np.array_equal(got[:, :, 0], exp["key"]) and np.array_equal(got[:, :, 1], exp["ref"]))
            ts = []
            for _ in range(a.reps):
                work.copy_(items)
                torch.cuda._sleep(200_000)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                backend.run_sorter_many(spec, work)
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e))
            ts.sort()
            ms = ts[len(ts) // 2]
            print(json.dumps({"n": n, "dist": dist, "ms": round(ms, 4),
                              "gbs": round(2 * a.rows * n * 16 / (ms / 1e3) / 1e9, 1), "ok": ok}), flush=True)


if __name__ == "__main__":
    main()
