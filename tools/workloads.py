"""Time every BASELINE configuration on one GPU (profiling companion of bench.py).

    python tools/workloads.py [--which cfg1,cfg2s,cfg3,cfg4,cfg5] [--reps 10]

Each workload: seeded synthetic inputs resident in HBM, W warm-up launches,
R timed launches with CUDA events on the launching stream (L2 flushed between
reps for cfg1, whose 64 MiB working set fits in L2), achieved GB/s against the
measured HBM peak, and a parity spot-check against the oracle.  Prints one
JSON object per workload.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def timeit(torch, fn, reps, warmup=3, flush=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        if flush is not None:
            flush()
        else:
            # keep the GPU busy while the host enqueues the timed launch, so
            # the start event does not absorb the Python call overhead
            torch.cuda._sleep(200_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return float(np.median(times)), float(np.min(times))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="cfg1,cfg3,cfg4,cfg5")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cfg5-rows", type=int, default=1 << 28)
    a = ap.parse_args()
    import torch

    import oracle
    from paper_2002_05599_b200 import batch
    dev = torch.device("cuda")
    pk = peak()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros(64 << 20, dtype=torch.float32, device=dev)

    def flush():
        # write 256 MiB (evicts the working set), then read 256 MiB so the L2
        # holds clean unrelated lines: the timed launch neither hits in L2
        # nor pays the write-back of the flush's dirty lines
        flush_buf.zero_()
        flush_rd.sum()

    out = []

    def report(name, nbytes, arrays, med, best, extra=None):
        rec = {"workload": name, "ms_median": round(med, 4), "ms_best": round(best, 4),
               "arrays_per_s": arrays / (med / 1e3), "gbs": round(nbytes / (med / 1e3) / 1e9, 1),
               "frac_of_measured_peak": round(nbytes / (med / 1e3) / 1e9 / pk, 4), "bytes": nbytes}
        rec.update(extra or {})
        out.append(rec)
        print(json.dumps(rec), flush=True)

    which = a.which.split(",")
    if "cfg1" in which:
        rows = 1 << 20
        keys = oracle.splitmix(rows * 8, seed=1, elem_bytes=4).reshape(rows, 8)
        kt = torch.from_numpy(keys.view(np.int32)).to(dev).view(torch.uint32)
        ot = torch.empty_like(kt)
        med, best = timeit(torch, lambda: batch.sort_rows(kt, out_keys=ot), a.reps, flush=flush)
        assert np.array_equal(ot.cpu().numpy(), np.sort(keys, axis=1))
        report("cfg1 2^20 x n=8 u32 best_08 (cold L2)", 2 * rows * 8 * 4, rows, med, best)
        med, best = timeit(torch, lambda: batch.sort_rows(kt, out_keys=ot), a.reps)
        report("cfg1 2^20 x n=8 u32 best_08 (warm L2, informational)", 2 * rows * 8 * 4, rows, med, best)

    if "cfg3" in which:
        rows = 1 << 20
        for n in (32, 64, 128, 256):
            g = torch.Generator(device=dev).manual_seed(n)
            uni = torch.randint(-2**63, 2**63 - 1, (rows, n), dtype=torch.int64, device=dev, generator=g)
            vals = torch.randint(-2**63, 2**63 - 1, (16,), dtype=torch.int64, device=dev, generator=g)
            few = vals[torch.randint(0, 16, (rows, n), device=dev, generator=g)]
            srt = torch.sort(uni, dim=1).values
            rev = torch.flip(srt, dims=[1]).contiguous()
            ot = torch.empty_like(uni)
            for dname, x in (("uniform", uni), ("few16", few), ("sorted", srt), ("reverse", rev)):
                for kind in ("rss", "merge"):
                    med, best = timeit(torch, lambda: batch.sort_rows(x, kind=kind, out_keys=ot), a.reps)
                    assert torch.equal(ot, torch.sort(x, dim=1).values)
                    label = "RSS 332" if kind == "rss" else "merge"
                    report(f"cfg3 {label} 2^20 x n={n} i64 {dname}", 2 * rows * n * 8, rows, med, best)
            del uni, few, srt, rev, ot
            torch.cuda.empty_cache()

    if "cfg4" in which:
        nseg = 67_108_864
        lengths = oracle.geometric_lengths(nseg, seed=4)
        off = np.zeros(nseg + 1, dtype=np.uint32)
        np.cumsum(lengths, out=off[1:])
        e = int(off[-1])
        u = oracle.splitmix(e, seed=40)
        w = ((u >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)
        ids = (u & np.uint64((1 << 26) - 1)).astype(np.uint32)
        ot = torch.from_numpy(off.view(np.int32)).to(dev).view(torch.uint32)
        wt = torch.from_numpy(w).to(dev)
        it = torch.from_numpy(ids.view(np.int32)).to(dev).view(torch.uint32)
        wo, io = torch.empty_like(wt), torch.empty_like(it)
        from paper_2002_05599_b200 import _lib
        ws = torch.empty(int(_lib.load_library().nsg_segments_ws_bytes(nseg, e)), dtype=torch.uint8, device=dev)
        fn = lambda: batch.sort_segments(ot, wt, it, descending=True, tie="unique", out_keys=wo, check=False,  # noqa: E731,E501
                                         out_payload=io, workspace=ws)
        med, best = timeit(torch, fn, a.reps)
        lo, hi = 2_000_000, 2_020_000
        sub = (off[lo:hi + 1] - off[lo]).astype(np.uint32)
        ek, ep = oracle.typed_sort_segments(sub, w[off[lo]:off[hi]], ids[off[lo]:off[hi]], descending=True)
        assert np.array_equal(wo[off[lo]:off[hi]].cpu().numpy(), ek)
        report("cfg4 CSR 67,108,864 segments f32 desc + u32 id", 2 * e * 8, nseg, med, best,
               {"elements": e, "offsets_bytes_not_counted": 4 * (nseg + 1),
                "elements_per_s": e / (med / 1e3)})

    if "cfg5" in which:
        rows = a.cfg5_rows
        from paper_2002_05599_b200 import _lib
        lib = _lib.lib()
        kt = torch.empty(rows * 16, dtype=torch.int64, device=dev)
        _lib.check(lib.nsg_fill_splitmix(kt.data_ptr(), rows * 16, 8, 5, 0, _lib.current_stream_handle()))
        kt = kt.view(torch.uint64).view(rows, 16)
        pt = torch.arange(rows * 16, dtype=torch.int64, device=dev).view(torch.uint64).view(rows, 16)
        ko, po = torch.empty_like(kt), torch.empty_like(pt)
        med, best = timeit(torch, lambda: batch.sort_rows(kt, pt, out_keys=ko, out_payload=po), max(3, a.reps // 2))
        sub_k = kt[:4096].cpu().numpy()
        sub_p = pt[:4096].cpu().numpy()
        ek, ep = oracle.typed_sort_rows(sub_k, sub_p)
        assert np.array_equal(ko[:4096].cpu().numpy(), ek) and np.array_equal(po[:4096].cpu().numpy(), ep)
        report(f"cfg5 {rows} x n=16 u64 key + u64 index, best_16 UNIQUE (1 GPU)", 2 * rows * 16 * 16, rows,
               med, best)
    return out


if __name__ == "__main__":
    main()
