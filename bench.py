#!/usr/bin/env python
"""Benchmark of the batched small-set sorter on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], "cfg2"): for every n = 2..16, a batch of
2^24 arrays of n uint64 keys (uniform, seeded counter-based generator), sorted
ascending with the best-known AND the Bose-Nelson network, both keys-only and
with a uint32 payload (= in-array index) compared lexicographically
(key, payload).  One STEP = all 60 (n, network, variant) launches = 1.007e9
sorted arrays.  At N GPUs every rank owns its own contiguous 2^24-array range
of an N*2^24-array global batch per cell (weak scaling, no collective on the
data path; one all-reduce of timings only).

Reported:
  value        whole-job sorted arrays/s, device-resident inputs, CUDA events,
               max over ranks;
  roofline     dominant kernel's achieved GB/s (algorithmic bytes = one read
               + one write of keys and payloads) vs measured HBM peak;
  e2e          same metric through the public API with HOST (pinned) buffers,
               host<->device copies inside the timed region;
  cpu_baseline the reference's own C core (oracle/_ref) on a bounded sample,
               all host threads (rank 0, N=1 only).
`--impl reference` times the reference's CPU path alone on the same sample.
Other workloads (--workload cfg1|cfg3|cfg4|cfg5) are for profiling; the driver
uses the default.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ROWS_CFG2 = 1 << 24
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg5"])
    ap.add_argument("--rows", type=int, default=None, help="override rows per cell (profiling)")
    ap.add_argument("--ns", default=None, help="comma list of n (profiling subset)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=1 << 17, help="CPU sample rows per cell")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# cells
# ---------------------------------------------------------------------------

class Cell:
    def __init__(self, name, n, family, key_bytes, pay_bytes, rows, unique=True, key_dtype="uint64",
                 pay_dtype=None):
        self.name, self.n, self.family = name, n, family
        self.kb, self.pb, self.rows = key_bytes, pay_bytes, rows
        self.unique, self.key_dtype, self.pay_dtype = unique, key_dtype, pay_dtype

    @property
    def bytes(self) -> int:  # algorithmic: one read + one write of keys and payloads
        return 2 * self.rows * self.n * (self.kb + self.pb)

    @property
    def kernel_key(self) -> str:  # name used by tools/profile_summary.py / profiles/traffic.json
        fam = "best" if self.family == "best" else "bn"
        pay = {0: "keys", 4: "p32", 8: "p64"}[self.pb]
        # rows of <= 64 bytes per region run the register-direct kernel
        # (net_direct_kernel, csrc/net_sort.cuh direct_row_ok)
        ok = lambda r: r <= 16 or r == 24 or (r % 16 == 0 and r <= 64)  # noqa: E731
        direct = ok(self.n * self.kb) and (self.pb == 0 or ok(self.n * self.pb))
        kind = "net_direct" if direct else "net_sort"
        return f"{kind} n={self.n} {fam} {'u64' if self.kb == 8 else 'u32'} {pay} SoA UNIQUE"


def make_cells(args, rows):
    ns = [int(x) for x in args.ns.split(",")] if args.ns else list(range(2, 17))
    cells = []
    if args.workload == "cfg2":
        for n in ns:
            for fam in ("best", "bn-l"):
                cells.append(Cell(f"n{n}_{fam}_keys", n, fam, 8, 0, rows))
                cells.append(Cell(f"n{n}_{fam}_kp32", n, fam, 8, 4, rows, pay_dtype="uint32"))
    elif args.workload == "cfg1":
        cells.append(Cell("n8_best_u32", 8, "best", 4, 0, rows, key_dtype="uint32"))
    elif args.workload == "cfg5":
        cells.append(Cell("n16_best_kp64", 16, "best", 8, 8, rows, pay_dtype="uint64"))
    return cells


def default_rows(workload):
    return {"cfg1": 1 << 20, "cfg2": ROWS_CFG2, "cfg5": 1 << 28}[workload]


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_for(kernel_name):
    """DRAM bytes per launch from the committed ncu --set full summary, if any."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel_name)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU legs (reference binary / oracle port) -- bounded samples
# ---------------------------------------------------------------------------

def cpu_sample_run(cells, sample_rows, threads):
    """Time the reference's own C core over `sample_rows` rows of every cell."""
    import oracle
    use_ref = oracle.ref_lib() is not None
    kind = "reference" if use_ref else "port"
    total_arrays, total_t = 0, 0.0
    for c in cells:
        rows = min(sample_rows, c.rows)
        keys = oracle.splitmix(rows * c.n, seed=0xC0FFEE + c.n, elem_bytes=c.kb).reshape(rows, c.n)
        items = np.empty((rows, c.n), dtype=oracle.ITEM)
        items["key"] = keys.astype(np.uint64)
        items["ref"] = np.broadcast_to(np.arange(c.n, dtype=np.uint64), (rows, c.n)) if c.pb else 0
        fam_code = ("best", "bn-l", "bn-p", "bn-r").index(c.family)
        spec = (0, fam_code, 5, 0, 0, 3, 3, 16, 0x5EED, 0, 16, 2, 0, 5)
        t0 = time.perf_counter()
        if use_ref:
            oracle.ref_run_items(items, spec, threads=threads)
        else:
            oracle.run_items(items, kind="network", family=c.family, unique=bool(c.pb), threads=threads)
        total_t += time.perf_counter() - t0
        total_arrays += rows
    return total_arrays / total_t, kind, total_arrays


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    rows = args.rows or default_rows(args.workload)
    cells = make_cells(args, rows)
    threads = oracle.cpu_count()
    sample = min(args.cpu_rows, rows)
    for _ in range(args.warmup):
        cpu_sample_run(cells, max(1, sample // 8), threads)
    vals, kind, arrays = [], None, 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, kind, arrays = cpu_sample_run(cells, sample, threads)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = float(np.median(vals))
    desc = (f"{sample} rows per cell x {len(cells)} cells of workload {args.workload} "
            f"({arrays} arrays per step), AoS (u64 key, u64 ref) items, ns_run_sorter per row")
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "arrays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (splitmix64 counter-based, seeded)",
        "config": config_block(args, rows, cells),
        "cpu_baseline": {"value": value, "unit": "arrays/s", "cores": threads, "kind": kind,
                         "sample": desc, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "arrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(args):
    return "sorted arrays/sec (and achieved HBM GB/s vs peak)"


def config_block(args, rows, cells):
    return {"workload": {"cfg1": "cfg1: 2^20 x n=8 uint32 keys, best_08",
                         "cfg2": "cfg2: n=2..16 x 2^24 arrays, uint64 keys, best + Bose-Nelson, "
                                 "keys-only and key+u32 payload (lexicographic)",
                         "cfg5": "cfg5 shard: n=16 uint64 key + uint64 payload, best_16"}[args.workload],
            "rows_per_cell": rows, "cells": len(cells), "ns": sorted({c.n for c in cells}),
            "l2": "inputs larger than L2 (smallest launch reads 256 MiB > 126 MB L2); no flush"}


# ---------------------------------------------------------------------------
# device leg
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2002_05599_b200 import _lib, batch, registry
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sh = int(stream.cuda_stream)

    rows = args.rows or default_rows(args.workload)
    cells = make_cells(args, rows)

    # inputs: one buffer per (n, variant); outputs shared (max size)
    inputs = {}
    max_k = max(c.rows * c.n * c.kb for c in cells)
    max_p = max(c.rows * c.n * max(c.pb, 1) for c in cells)
    out_k = torch.empty(max_k, dtype=torch.uint8, device=dev)
    out_p = torch.empty(max_p, dtype=torch.uint8, device=dev)
    for c in cells:
        key = (c.n, c.kb, c.pb)
        if key in inputs:
            continue
        kbuf = torch.empty(c.rows * c.n * c.kb, dtype=torch.uint8, device=dev)
        first = rank * c.rows * c.n
        _lib.check(lib.nsg_fill_splitmix(kbuf.data_ptr(), c.rows * c.n, c.kb, 0xC0FFEE + c.n, first, sh))
        pbuf = None
        if c.pb:
            pbuf = torch.arange(c.n, dtype=torch.int32 if c.pb == 4 else torch.int64,
                                device=dev).repeat(c.rows).view(torch.uint8)
        inputs[key] = (kbuf, pbuf)
    torch.cuda.synchronize(dev)

    specs = {}
    for c in cells:
        order = registry.DeviceOrder(registry.KEY_DTYPES[c.key_dtype],
                                     registry.PAY_DTYPES[c.pay_dtype], 0,
                                     registry.TIE_UNIQUE if c.unique else registry.TIE_REF)
        specs[c.name] = _lib.make_spec(registry.spec_network(c.family, "4CmS"), order)

    def launch(c):
        kbuf, pbuf = inputs[(c.n, c.kb, c.pb)]
        rc = lib.nsg_sort_rows(specs[c.name], kbuf.data_ptr(), out_k.data_ptr(),
                               pbuf.data_ptr() if pbuf is not None else None,
                               out_p.data_ptr() if pbuf is not None else None, c.rows, c.n, sh)
        if rc:
            _lib.check(rc)

    for _ in range(args.warmup):
        for c in cells:
            launch(c)
    torch.cuda.synchronize(dev)

    # correctness of this run: re-run every distinct (n, variant) and check a prefix on the device
    verify(cells, inputs, out_k, out_p, launch, dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps * len(cells))]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        i = 0
        for _ in range(args.steps):
            for c in cells:
                ev[i][0].record(stream)
                launch(c)
                ev[i][1].record(stream)
                i += 1
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    per_cell = {c.name: 0.0 for c in cells}
    i = 0
    for _ in range(args.steps):
        for c in cells:
            per_cell[c.name] += ev[i][0].elapsed_time(ev[i][1])
            i += 1
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())

    arrays_per_step = sum(c.rows for c in cells)
    bytes_per_step = sum(c.bytes for c in cells)
    value = world * arrays_per_step * args.steps / (elapsed_ms / 1e3)
    peak, peak_src = hbm_peak()
    dom = max(cells, key=lambda c: per_cell[c.name])
    dom_ms = per_cell[dom.name] / args.steps
    achieved = dom.bytes / (dom_ms / 1e3) / 1e9
    kern_total_ms = sum(per_cell.values()) / args.steps
    agg_gbs = bytes_per_step / (kern_total_ms / 1e3) / 1e9

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(cells, batch, dev, world, rank, steps=max(1, min(args.steps, 2)))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        threads = oracle.cpu_count()
        sample = min(args.cpu_rows, rows)
        v, kind, arrays = cpu_sample_run(cells, sample, threads)
        cpu = {"value": v, "unit": "arrays/s", "cores": threads, "kind": kind, "cpu": cpu_model(),
               "sample": f"{sample} rows per cell x {len(cells)} cells ({arrays} arrays), "
                         "AoS (u64 key, u64 ref) items, reference ns_run_sorter row loop over all host threads"}

    if rank == 0:
        per_kernel = {c.name: round(c.bytes / (per_cell[c.name] / args.steps / 1e3) / 1e9, 1) for c in cells}
        line = {
            "metric": metric_name(args), "value": value, "unit": "arrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (splitmix64 counter-based, seeded, keyed by global element index)",
            "config": config_block(args, rows, cells),
            "elements_per_s": world * sum(c.rows * c.n for c in cells) * args.steps / (elapsed_ms / 1e3),
            "hbm_gbs_aggregate": round(agg_gbs, 1),
            "hbm_frac_aggregate": round(agg_gbs / peak, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic_for(dom.kernel_key),
                         "traffic_source": "profiles/traffic.json (ncu --set full dram__bytes_read+write per launch)",
                         "kernel": dom.kernel_key, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": dom.bytes, "avg_launch_ms": round(dom_ms, 4)},
            "per_kernel_gbs": per_kernel,
            "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": len(cells) * args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def verify(cells, inputs, out_k, out_p, launch, dev):
    import torch

    import oracle
    seen = set()
    for c in cells:
        key = (c.n, c.kb, c.pb, c.family)
        if key in seen:
            continue
        seen.add(key)
        launch(c)
        torch.cuda.synchronize(dev)
        m = min(c.rows, 2048)
        kbuf, pbuf = inputs[(c.n, c.kb, c.pb)]
        kd = np.uint64 if c.kb == 8 else np.uint32
        keys_in = kbuf[: m * c.n * c.kb].cpu().numpy().view(kd).reshape(m, c.n)
        got_k = out_k[: m * c.n * c.kb].cpu().numpy().view(kd).reshape(m, c.n)
        pay_in = got_p = None
        if c.pb:
            pd = np.uint32 if c.pb == 4 else np.uint64
            pay_in = pbuf[: m * c.n * c.pb].cpu().numpy().view(pd).reshape(m, c.n)
            got_p = out_p[: m * c.n * c.pb].cpu().numpy().view(pd).reshape(m, c.n)
        ek, ep = oracle.typed_sort_rows(keys_in, pay_in, family=c.family, unique=c.unique)
        from paper_2002_05599_b200.errors import CorrectnessFailure
        if not np.array_equal(ek, got_k) or (c.pb and not np.array_equal(ep, got_p)):
            raise CorrectnessFailure(f"bench verification failed for {c.name} (oracle prefix)")
        # every row of the launch: ordered + permutation of its input, on device
        bad = verify_device(c, kbuf, pbuf, out_k, out_p, dev)
        if bad:
            raise CorrectnessFailure(f"bench verification failed for {c.name}: {bad} bad rows (device check)")


def verify_device(c, kbuf, pbuf, out_k, out_p, dev) -> int:
    import torch

    from paper_2002_05599_b200 import _lib, registry
    order = registry.DeviceOrder(registry.KEY_DTYPES[c.key_dtype], registry.PAY_DTYPES[c.pay_dtype], 0,
                                 registry.TIE_UNIQUE if c.unique else registry.TIE_REF)
    sp = _lib.make_spec(registry.spec_network(c.family, "4CmS"), order)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().nsg_verify_rows(sp, kbuf.data_ptr(), pbuf.data_ptr() if pbuf is not None else None,
                                          out_k.data_ptr(), out_p.data_ptr() if pbuf is not None else None,
                                          c.rows, c.n, bad.data_ptr(), _lib.current_stream_handle(dev)))
    return int(bad.item())


def run_e2e(cells, batch, dev, world, rank, steps):
    import torch
    import torch.distributed as dist

    import oracle
    max_rows = max(c.rows for c in cells)
    max_n = max(c.n for c in cells)
    hk = torch.empty(max_rows * max_n, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    hk[:] = oracle.splitmix(max_rows * max_n, seed=0xE2E + rank)
    hp = torch.empty(max_rows * max_n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    hp[:] = np.tile(np.arange(max_n, dtype=np.uint32), max_rows)
    ok = torch.empty(max_rows * max_n, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    op = torch.empty(max_rows * max_n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    h2d = d2h = 0
    arrays = 0

    def one_step():
        nonlocal h2d, d2h, arrays
        h2d = d2h = arrays = 0
        for c in cells:
            k = hk[: c.rows * c.n].reshape(c.rows, c.n)
            p = hp[: c.rows * c.n].reshape(c.rows, c.n) if c.pb else None
            batch.sort_rows(k, p, family=c.family, tie="unique" if c.unique else "ref",
                            out_keys=ok[: c.rows * c.n].reshape(c.rows, c.n),
                            out_payload=op[: c.rows * c.n].reshape(c.rows, c.n) if c.pb else None)
            h2d += k.nbytes + (p.nbytes if p is not None else 0)
            d2h += k.nbytes + (p.nbytes if p is not None else 0)
            arrays += c.rows

    one_step()  # warm-up (allocates the library's staging buffers)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": world * arrays * steps / dt, "unit": "arrays/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "path": "batch.sort_rows(numpy pinned) -> nsg_sort_rows_host (chunked H2D/sort/D2H, 3 streams)"}


if __name__ == "__main__":
    main()
