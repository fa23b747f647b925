"""Time the row sorters on BASELINE cfg3 shapes (2^20 rows x n int64, four
distributions) and check each output against torch.sort.

    python tools/cfg3_probe.py [--ns 32,64,128,256] [--kinds merge,rss] [--reps 10]

One JSON line per (kind, n, distribution): median ms, GB/s (one read + one
write of the keys) and the fraction of the measured HBM peak, plus the
packed-key kernels' exact-fallback row count.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="32,64,128,256")
    ap.add_argument("--kinds", default="merge,rss")
    ap.add_argument("--dists", default="uniform,few16,sorted,reverse")
    ap.add_argument("--rows", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_2002_05599_b200 import batch
    from paper_2002_05599_b200._lib import lib
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6650.0
    dev = torch.device("cuda")
    for n in [int(x) for x in a.ns.split(",")]:
        g = torch.Generator(device=dev).manual_seed(n)
        uni = torch.randint(-2**63, 2**63 - 1, (a.rows, n), dtype=torch.int64, device=dev, generator=g)
        data = {}
        for d in a.dists.split(","):
            if d == "uniform":
                data[d] = uni
            elif d == "few16":
                vals = torch.randint(-2**63, 2**63 - 1, (16,), dtype=torch.int64, device=dev, generator=g)
                data[d] = vals[torch.randint(0, 16, (a.rows, n), device=dev, generator=g)]
            elif d == "sorted":
                data[d] = torch.sort(uni, dim=1).values
            elif d == "reverse":
                data[d] = torch.flip(torch.sort(uni, dim=1).values, dims=[1]).contiguous()
        for d, x in data.items():
            exp = torch.sort(x, dim=1).values
            for kind in a.kinds.split(","):
                out = torch.empty_like(x)
                lib().nsg_rss_fallback_rows(1)
                batch.sort_rows(x, kind=kind, out_keys=out)
                torch.cuda.synchronize()
                fb = int(lib().nsg_rss_fallback_rows(1))
                ok = bool(torch.equal(out, exp))
                for _ in range(3):
                    batch.sort_rows(x, kind=kind, out_keys=out)
                ts = []
                for _ in range(a.reps):
                    torch.cuda._sleep(100_000)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    batch.sort_rows(x, kind=kind, out_keys=out)
                    e.record()
                    e.synchronize()
                    ts.append(s.elapsed_time(e))
                ts.sort()
                ms = ts[len(ts) // 2]
                gbs = 2 * x.numel() * 8 / (ms / 1e3) / 1e9
                print(json.dumps({"kind": kind, "n": n, "dist": d, "ms": round(ms, 4), "gbs": round(gbs, 1),
                                  "frac": round(gbs / pk, 4), "ok": ok, "fallback_rows": fb}), flush=True)


if __name__ == "__main__":
    main()
