#!/usr/bin/env python
"""Benchmark of the batched small-set sorter on B200 (one JSON line on rank 0).

Headline (`value`, BASELINE.json configs[1], "cfg2"): for every n = 2..16, a
batch of 2^24 arrays of n uint64 keys (uniform, seeded counter-based
generator), sorted ascending with the best-known AND the Bose-Nelson network,
both keys-only and with a uint32 payload (= in-array index) compared
lexicographically (key, payload).  One STEP = all 60 (n, network, variant)
launches = 1.007e9 sorted arrays.  At N GPUs every rank owns its own
contiguous 2^24-array range of an N*2^24-array global batch per cell (weak
scaling, no collective on the data path).

The same JSON line carries one verified, CUDA-event-timed block per other
BASELINE configuration under "workloads" (default `--workloads all`):
  cfg1  2^20 x n=8 uint32, best_08, L2 flushed between reps; a same-box
        device copy of the same bytes is timed beside it as the ceiling;
  cfg3  Register Sample Sort 332 (and the merge sorter) x {uniform, few16,
        sorted, reverse} x n in {32, 64, 128, 256}, 2^20 int64 rows each, plus
        the reference-shaped entry (run_sorter_many on AoS (key, ref) items,
        REF mode) on the uniform rows;
  cfg4  67,108,864 CSR segments (truncated geometric lengths 1..16), f32
        weights descending + u32 ids;
  cfg5  2^28 arrays of 16 uint64 keys + uint64 global index, best_16 UNIQUE,
        the 2^28 arrays SPLIT across the N ranks (strong scaling), per-GPU and
        aggregate GB/s.
Every block is checked against the CPU oracle on a prefix and on the device
for every row/segment (order + multiset).

Reported:
  value        whole-job sorted arrays/s (cfg2), device-resident inputs, CUDA
               events, max over ranks;
  roofline     dominant cfg2 kernel's achieved GB/s (algorithmic bytes = one
               read + one write of keys and payloads) vs measured HBM peak;
  e2e          same metric through the public API with HOST (pinned) buffers,
               host<->device copies inside the timed region, outputs checked;
  cpu_baseline the reference's own C core (oracle/_ref) on a bounded,
               cache-cold sample, at T = all host threads and at T = 1
               (rank 0, N = 1 only).
`--impl reference` times the reference's CPU path alone on the same sample.
Multi-rank plumbing (barriers, max-over-ranks) uses a gloo process group: the
path has no collective, NCCL is not used.
"""

from __future__ import annotations

import argparse
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
WORKLOADS = ("cfg1", "cfg3", "cfg4", "cfg5")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg5"],
                    help="headline workload (profiling: cfg1/cfg5 as the timed step)")
    ap.add_argument("--workloads", default="all",
                    help="extra verified blocks: all | none | comma list of cfg1,cfg3,cfg4,cfg5")
    ap.add_argument("--rows", type=int, default=None, help="override rows per cell (profiling)")
    ap.add_argument("--ns", default=None, help="comma list of n (profiling subset)")
    ap.add_argument("--cfg5-rows", type=int, default=1 << 28)
    ap.add_argument("--cfg3-ns", default="32,64,128,256")
    ap.add_argument("--reps", type=int, default=10, help="timed reps per workload block")
    ap.add_argument("--dump-dir", default=None, help="write each rank's cfg5 shard digest here (tests)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=1 << 17, help="CPU sample rows per cell")
    return ap.parse_args()


def workload_list(args):
    if args.workloads in ("", "none"):
        return []
    if args.workloads == "all":
        return list(WORKLOADS)
    w = [x.strip() for x in args.workloads.split(",") if x.strip()]
    for x in w:
        if x not in WORKLOADS:
            raise SystemExit(f"unknown workload {x}")
    return w


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
        kt = "u64" if self.kb == 8 else "u32"
        # staged by TMA (mirrors csrc/capi.cu dispatch: nettma_covers, netbulk.cu nb_choice)
        if self.kb == 8 and self.n == 16 and self.pb == 4:
            return f"nettma n=16 {fam} {kt} {pay} SoA UNIQUE"
        if self.kb == 8 and self.pb in (0, 4) and self.n % 2 and 5 <= self.n <= 15:
            d = 0 if self.family == "best" else 1
            bulk = (self.n in (5, 7, 11, 13) or (self.n == 15 and d == 0)) if self.pb == 0 else \
                (self.n in (9, 11) or (self.n == 13 and d == 0) or self.n == 15)
            if bulk:
                return f"netbulk n={self.n} {fam} {kt} {pay} SoA UNIQUE"
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
    return {"cfg1": 1 << 20, "cfg2": ROWS_CFG2, "cfg5": 1 << 24}[workload]


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


def cpu_info():
    model, mhz = "unknown", []
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
            elif line.startswith("cpu MHz"):
                mhz.append(float(line.split(":", 1)[1]))
    except OSError:
        pass
    return {"cpu": model, "cpu_mhz_median": round(float(np.median(mhz)), 1) if mhz else None}


# ---------------------------------------------------------------------------
# distributed plumbing: gloo (host) only -- the sort path has no collective
# ---------------------------------------------------------------------------

class Group:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not self.dist:
            return float(v)
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, v: float) -> list:
        if not self.dist:
            return [float(v)]
        import torch
        out = [torch.zeros(1, dtype=torch.float64) for _ in range(self.world)]
        self.dist.all_gather(out, torch.tensor([float(v)], dtype=torch.float64))
        return [float(x.item()) for x in out]

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU legs (reference binary / oracle port) -- bounded, cache-cold samples
# ---------------------------------------------------------------------------

def _net_spec(family):
    fam_code = ("best", "bn-l", "bn-p", "bn-r").index(family)
    return (0, fam_code, 5, 0, 0, 3, 3, 16, 0x5EED, 0, 16, 2, 0, 5)


RSS332_SPEC = (2, 0, 5, 0, 0, 3, 3, 16, 0x5EED, 0, 16, 2, 0, 5)


def _cpu_run(items, spec, threads, family="best", kind="network", unique=False):
    import oracle
    if oracle.ref_lib() is not None:
        oracle.ref_run_items(items, spec, threads=threads)
        return "reference"
    oracle.run_items(items, kind=kind, family=family, unique=unique, threads=threads)
    return "port"


def cpu_cells_samples(cells, sample_rows):
    """Per-cell AoS item samples, ALL generated before any timing: the ~1 GB of
    other cells' rows written since a cell's sample was made evicts it from
    the LLC, so every timed cell starts cache-cold."""
    import oracle
    out = []
    for c in cells:
        rows = min(sample_rows, c.rows)
        keys = oracle.splitmix(rows * c.n, seed=0xC0FFEE + c.n, elem_bytes=c.kb).reshape(rows, c.n)
        items = np.empty((rows, c.n), dtype=oracle.ITEM)
        items["key"] = keys.astype(np.uint64)
        items["ref"] = np.broadcast_to(np.arange(c.n, dtype=np.uint64), (rows, c.n)) if c.pb else 0
        out.append(items)
    return out


def cpu_sample_run(cells, samples, threads):
    total_arrays, total_t, kind = 0, 0.0, None
    for c, items in zip(cells, samples):
        t0 = time.perf_counter()
        kind = _cpu_run(items, _net_spec(c.family), threads, family=c.family, unique=bool(c.pb))
        total_t += time.perf_counter() - t0
        total_arrays += items.shape[0]
    return total_arrays / total_t, kind, total_arrays


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    rows = args.rows or default_rows(args.workload)
    cells = make_cells(args, rows)
    threads = oracle.cpu_count()
    sample = min(args.cpu_rows, rows)
    samples = cpu_cells_samples(cells, sample)
    for _ in range(args.warmup):
        cpu_sample_run(cells, [s[: max(1, s.shape[0] // 8)] for s in samples], threads)
    vals, kind, arrays = [], None, 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, kind, arrays = cpu_sample_run(cells, samples, threads)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = float(np.median(vals))
    desc = (f"{sample} rows per cell x {len(cells)} cells of workload {args.workload} "
            f"({arrays} arrays per step, cache-cold), AoS (u64 key, u64 ref) items, ns_run_sorter per row "
            f"on {threads} threads over contiguous row slices")
    cfg = config_block(args, rows, cells)
    cfg["rows_per_cell"] = sample
    cfg["rows_per_cell_note"] = f"CPU sample of the {rows}-row cells (throughput is size-independent past the LLC)"
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "arrays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (splitmix64 counter-based, seeded)",
        "config": cfg,
        "cpu_baseline": dict({"value": value, "unit": "arrays/s", "cores": threads, "kind": kind,
                              "sample": desc}, **cpu_info()),
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
# device helpers
# ---------------------------------------------------------------------------

def ev_time(torch, fn, reps, warmup=2, flush=None):
    """Median and best of `reps` launches of fn, CUDA events on the current stream."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        if flush is not None:
            flush()
        else:
            torch.cuda._sleep(200_000)  # keep the GPU busy while the host enqueues fn
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return float(np.median(times)), float(np.min(times))


def rate_block(nbytes, arrays, elements, med, best, peak):
    gbs = nbytes / (med / 1e3) / 1e9
    return {"ms_median": round(med, 4), "ms_best": round(best, 4), "arrays_per_s": arrays / (med / 1e3),
            "elements_per_s": elements / (med / 1e3), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
            "bytes": int(nbytes)}


def device_bad_rows(lib, _lib, registry, kin, pin, kout, pout, rows, n, key_dtype, pay_dtype, descending=False,
                    unique=True, dev=None):
    import torch
    order = registry.DeviceOrder(registry.KEY_DTYPES[key_dtype], registry.PAY_DTYPES[pay_dtype],
                                 int(descending), registry.TIE_UNIQUE if unique else registry.TIE_REF)
    sp = _lib.make_spec(registry.spec_network("best", "4CmS"), order)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(lib.nsg_verify_rows(sp, kin.data_ptr(), pin.data_ptr() if pin is not None else None,
                                   kout.data_ptr(), pout.data_ptr() if pout is not None else None, rows, n,
                                   bad.data_ptr(), _lib.current_stream_handle(dev)))
    return int(bad.item())


# ---------------------------------------------------------------------------
# device leg: headline (cfg2)
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    from paper_2002_05599_b200 import _lib, batch, registry
    grp = Group()
    world, rank, local = grp.world, grp.rank, grp.local
    # one GPU per rank; more ranks than GPUs (the 2-rank GPU test on a 1-GPU
    # box) share devices -- safe here: no kernel waits on another rank
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sh = int(stream.cuda_stream)
    peak, peak_src = hbm_peak()

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

    # correctness of this run: re-run every distinct (n, variant) and check a prefix + every row
    verify(cells, inputs, out_k, out_p, launch, dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps * len(cells))]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    grp.barrier()
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
    grp.barrier()
    elapsed_ms = grp.max(t_start.elapsed_time(t_end))
    per_cell = {c.name: 0.0 for c in cells}
    i = 0
    for _ in range(args.steps):
        for c in cells:
            per_cell[c.name] += ev[i][0].elapsed_time(ev[i][1])
            i += 1

    arrays_per_step = sum(c.rows for c in cells)
    bytes_per_step = sum(c.bytes for c in cells)
    value = world * arrays_per_step * args.steps / (elapsed_ms / 1e3)
    dom = max(cells, key=lambda c: per_cell[c.name])
    dom_ms = per_cell[dom.name] / args.steps
    achieved = dom.bytes / (dom_ms / 1e3) / 1e9
    kern_total_ms = sum(per_cell.values()) / args.steps
    agg_gbs = bytes_per_step / (kern_total_ms / 1e3) / 1e9
    del ev

    # e2e through the public API with pinned host buffers (outputs checked)
    inputs.clear()
    del out_k, out_p
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(cells, batch, dev, grp, steps=max(1, min(args.steps, 2)))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_cfg2(args, cells, rows)

    # the other BASELINE configurations, one verified block each
    blocks = {}
    for w in workload_list(args):
        if w != "cfg5" and world > 1:
            continue  # N>1: only the strong-scaled cfg5 split is defined across ranks
        fn = {"cfg1": wl_cfg1, "cfg3": wl_cfg3, "cfg4": wl_cfg4, "cfg5": wl_cfg5}[w]
        blocks[w] = fn(args, torch, dev, grp, peak, want_cpu=(rank == 0 and world == 1 and not args.no_cpu))
        torch.cuda.empty_cache()

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
                         "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write per launch)",
                         "kernel": dom.kernel_key, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": dom.bytes, "avg_launch_ms": round(dom_ms, 4)},
            "per_kernel_gbs": per_kernel,
            "min_kernel_gbs": min(per_kernel.values()),
            "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": len(cells) * args.steps,
            "clocks": clocks.summary(),
            "workloads": blocks,
        }
        print(json.dumps(line), flush=True)
    grp.close()


def cpu_baseline_cfg2(args, cells, rows):
    import oracle
    threads = oracle.cpu_count()
    sample = min(args.cpu_rows, rows)
    samples = cpu_cells_samples(cells, sample)
    v, kind, arrays = cpu_sample_run(cells, samples, threads)
    s1 = max(1, sample // 8)
    samples1 = cpu_cells_samples(cells, s1)
    v1, _, arrays1 = cpu_sample_run(cells, samples1, 1)
    elem = sum(min(sample, c.rows) * c.n for c in cells)
    return dict({"value": v, "unit": "arrays/s", "cores": threads, "kind": kind,
                 "value_t1": v1, "cores_t1": 1,
                 "elements_per_s": v * elem / arrays,
                 "gbs": v * sum(2 * min(sample, c.rows) * c.n * (c.kb + c.pb) for c in cells) / arrays / 1e9,
                 "sample": f"{sample} rows per cell x {len(cells)} cells ({arrays} arrays) at T={threads}; "
                           f"{s1} rows per cell ({arrays1} arrays) at T=1; rows generated before timing "
                           "(cache-cold), AoS (u64 key, u64 ref) items, reference ns_run_sorter row loop "
                           "over contiguous row slices"}, **cpu_info())


def verify(cells, inputs, out_k, out_p, launch, dev):
    import torch

    import oracle
    from paper_2002_05599_b200 import _lib, registry
    from paper_2002_05599_b200.errors import CorrectnessFailure
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
        if not np.array_equal(ek, got_k) or (c.pb and not np.array_equal(ep, got_p)):
            raise CorrectnessFailure(f"bench verification failed for {c.name} (oracle prefix)")
        bad = device_bad_rows(_lib.lib(), _lib, registry, kbuf, pbuf, out_k, out_p if pbuf is not None else None,
                              c.rows, c.n, c.key_dtype, c.pay_dtype, unique=c.unique, dev=dev)
        if bad:
            raise CorrectnessFailure(f"bench verification failed for {c.name}: {bad} bad rows (device check)")


def run_e2e(cells, batch, dev, grp, steps):
    import torch

    import oracle
    from paper_2002_05599_b200.errors import CorrectnessFailure
    world, rank = grp.world, grp.rank
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

    def one_step(check=False):
        nonlocal h2d, d2h, arrays
        h2d = d2h = arrays = 0
        for c in cells:
            k = hk[: c.rows * c.n].reshape(c.rows, c.n)
            p = hp[: c.rows * c.n].reshape(c.rows, c.n) if c.pb else None
            okc = ok[: c.rows * c.n].reshape(c.rows, c.n)
            opc = op[: c.rows * c.n].reshape(c.rows, c.n) if c.pb else None
            batch.sort_rows(k, p, family=c.family, tie="unique" if c.unique else "ref", out_keys=okc,
                            out_payload=opc)
            h2d += k.nbytes + (p.nbytes if p is not None else 0)
            d2h += k.nbytes + (p.nbytes if p is not None else 0)
            arrays += c.rows
            if check:  # host output of this cell: oracle on a prefix (outside the timed steps)
                m = 512
                ek, ep = oracle.typed_sort_rows(k[:m], None if p is None else p[:m], family=c.family,
                                                unique=c.unique)
                if not np.array_equal(okc[:m], ek) or (p is not None and not np.array_equal(opc[:m], ep)):
                    raise CorrectnessFailure(f"e2e output mismatch for {c.name}")

    one_step(check=True)  # warm-up (allocates the library's staging buffers) + output check
    grp.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    dt = grp.max(time.perf_counter() - t0)
    # the timed steps' final output (last cell) is checked again
    c = cells[-1]
    m = 512
    k = hk[: c.rows * c.n].reshape(c.rows, c.n)[:m]
    p = hp[: c.rows * c.n].reshape(c.rows, c.n)[:m] if c.pb else None
    ek, ep = oracle.typed_sort_rows(k, p, family=c.family, unique=c.unique)
    if not np.array_equal(ok[: c.rows * c.n].reshape(c.rows, c.n)[:m], ek):
        raise CorrectnessFailure("e2e output mismatch after the timed steps")
    return {"value": world * arrays * steps / dt, "unit": "arrays/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "verified": "oracle prefix of every cell's host output",
            "path": "batch.sort_rows(numpy pinned) -> nsg_sort_rows_host (chunked H2D/sort/D2H, 3 streams)"}


# ---------------------------------------------------------------------------
# workload blocks (BASELINE configs[0], [2], [3], [4])
# ---------------------------------------------------------------------------

def wl_cfg1(args, torch, dev, grp, peak, want_cpu):
    import oracle
    from paper_2002_05599_b200 import batch
    from paper_2002_05599_b200.errors import CorrectnessFailure
    rows = 1 << 20
    keys = oracle.splitmix(rows * 8, seed=1, elem_bytes=4).reshape(rows, 8)
    kt = torch.from_numpy(keys.view(np.int32)).to(dev).view(torch.uint32)
    ot = torch.empty_like(kt)
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)

    def flush():  # evict the working set, leave clean unrelated lines in L2
        flush_w.zero_()
        flush_r.sum()

    med, best = ev_time(torch, lambda: batch.sort_rows(kt, out_keys=ot), args.reps, flush=flush)
    got = ot.cpu().numpy()
    ek, _ = oracle.typed_sort_rows(keys[:4096], family="best")
    if not np.array_equal(got[:4096], ek) or not np.array_equal(got, np.sort(keys, axis=1)):
        raise CorrectnessFailure("cfg1 verification failed")
    nbytes = 2 * rows * 8 * 4
    blk = rate_block(nbytes, rows, rows * 8, med, best, peak)
    blk.update({"workload": "cfg1: 2^20 x n=8 uint32, best_08 (19 comparators), L2 flushed between reps",
                "kernel": "net_direct n=8 best u32 keys SoA UNIQUE",
                "verified": "oracle on 4096 rows + np.sort on all rows"})
    # ceiling: a device copy of the same 32 MiB (64 MiB of traffic), same flush
    cp_med, cp_best = ev_time(torch, lambda: ot.copy_(kt), args.reps, flush=flush)
    blk["copy_ceiling"] = {"what": "torch copy_ of the same 32 MiB, L2 flushed", "ms_median": round(cp_med, 4),
                           "gbs": round(nbytes / (cp_med / 1e3) / 1e9, 1),
                           "sort_vs_copy": round(cp_med / med, 4)}
    med_w, _ = ev_time(torch, lambda: batch.sort_rows(kt, out_keys=ot), args.reps)
    blk["warm_l2_ms_median"] = round(med_w, 4)
    if want_cpu:
        items = np.empty((rows, 8), dtype=oracle.ITEM)
        items["key"] = keys.astype(np.uint64)
        items["ref"] = 0
        blk["cpu_baseline"] = cpu_block(items, _net_spec("best"), rows, nbytes, "all 2^20 rows")
    del flush_w, flush_r
    return blk


def cpu_block(items, spec, arrays, nbytes, what, kind="network", t1_rows=None):
    """Reference CPU core on `items` at T = all (and T = 1 on a prefix)."""
    import oracle
    threads = oracle.cpu_count()
    t0 = time.perf_counter()
    k = _cpu_run(items, spec, threads, kind=kind)
    dt = time.perf_counter() - t0
    out = {"arrays_per_s": items.shape[0] / dt, "gbs": nbytes * items.shape[0] / arrays / dt / 1e9,
           "cores": threads, "kind": k, "sample": what}
    m = t1_rows or max(1, items.shape[0] // 16)
    sub = np.ascontiguousarray(items[:m])
    t0 = time.perf_counter()
    _cpu_run(sub, spec, 1, kind=kind)
    out["arrays_per_s_t1"] = m / (time.perf_counter() - t0)
    return out


def cfg3_inputs(torch, dev, n, rows):
    g = torch.Generator(device=dev).manual_seed(n)
    uni = torch.randint(-2**63, 2**63 - 1, (rows, n), dtype=torch.int64, device=dev, generator=g)
    vals = torch.randint(-2**63, 2**63 - 1, (16,), dtype=torch.int64, device=dev, generator=g)
    few = vals[torch.randint(0, 16, (rows, n), device=dev, generator=g)]
    srt = torch.sort(uni, dim=1).values
    rev = torch.flip(srt, dims=[1]).contiguous()
    return (("uniform", uni), ("few16", few), ("sorted", srt), ("reverse", rev))


def cfg3_items_cell(torch, dev, x, n, rows, reps, peak):
    """run_sorter_many(spec_rss("332"), items) on device-resident reference items
    (16 bytes each: u64 key, u64 ref), checked against the oracle on 512 rows
    and for key order / ref permutation on all rows."""
    import oracle
    from paper_2002_05599_b200 import backend, registry
    from paper_2002_05599_b200.errors import CorrectnessFailure
    spec = registry.spec_rss("332")
    items = torch.empty((rows, n, 2), dtype=torch.int64, device=dev)
    items[:, :, 0] = x ^ (-2**63)
    items[:, :, 1] = torch.arange(rows * n, device=dev).view(rows, n)
    work = torch.empty_like(items)
    times = []
    for rep in range(reps + 2):
        work.copy_(items)
        torch.cuda._sleep(200_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        backend.run_sorter_many(spec, work)
        e.record()
        e.synchronize()
        if rep >= 2:
            times.append(s.elapsed_time(e))
    sub = items[:512].cpu().numpy().view(np.uint64)
    exp = np.empty((512, n), dtype=oracle.ITEM)
    exp["key"], exp["ref"] = sub[:, :, 0], sub[:, :, 1]
    oracle.run_items(exp, kind="rss", rss_cfg="332")
    got = work[:512].cpu().numpy().view(np.uint64)
    keys_u = work[:, :, 0] ^ (-2**63)  # back to int64 order
    ok = bool((keys_u[:, 1:] >= keys_u[:, :-1]).all())
    ok = ok and bool(torch.equal(torch.sort(work[:, :, 1], dim=1).values, items[:, :, 1]))
    if not ok or not (np.array_equal(got[:, :, 0], exp["key"]) and np.array_equal(got[:, :, 1], exp["ref"])):
        raise CorrectnessFailure(f"cfg3 items n={n}: parity")
    blk = rate_block(2 * rows * n * 16, rows, rows * n, float(np.median(times)), float(np.min(times)), peak)
    blk["api"] = "backend.run_sorter_many(spec_rss('332'), items) -- AoS (u64 key, u64 ref), REF mode, in place"
    del items, work
    return blk


def wl_cfg3(args, torch, dev, grp, peak, want_cpu):
    import oracle
    from paper_2002_05599_b200 import _lib, batch, registry
    from paper_2002_05599_b200.errors import CorrectnessFailure
    lib = _lib.lib()
    rows = 1 << 20
    res = {"workload": "cfg3: 2^20 x n int64 rows, RSS 332 (SN Best base) and the merge sorter",
           "verified": "oracle (reference RSS restatement) on 512 rows + device order/multiset check of all rows",
           "cells": {}}
    for n in [int(x) for x in args.cfg3_ns.split(",")]:
        ins = cfg3_inputs(torch, dev, n, rows)
        ot = torch.empty_like(ins[0][1])
        for dname, x in ins:
            for kind in ("rss", "merge"):
                med, best = ev_time(torch, lambda: batch.sort_rows(x, kind=kind, out_keys=ot), args.reps)
                bad = device_bad_rows(lib, _lib, registry, x, None, ot, None, rows, n, "int64", None, dev=dev)
                xs = x[:512].cpu().numpy()
                ek, _ = oracle.typed_sort_rows(xs, kind="rss")
                if bad or not np.array_equal(ot[:512].cpu().numpy(), ek):
                    raise CorrectnessFailure(f"cfg3 {kind} n={n} {dname}: {bad} bad rows")
                res["cells"][f"{'rss' if kind == 'rss' else 'merge'}_n{n}_{dname}"] = rate_block(
                    2 * rows * n * 8, rows, rows * n, med, best, peak)
        # the reference-shaped entry on the same uniform rows: run_sorter_many on
        # AoS (key ^ 2^63, ref = global index) items, RSS 332 in REF mode, in place
        res["cells"][f"rss_items_n{n}_uniform"] = cfg3_items_cell(torch, dev, ins[0][1], n, rows, args.reps, peak)
        if want_cpu:
            for dname, x in ins:
                m = {32: 32768, 64: 16384, 128: 8192, 256: 4096}.get(n, 4096)
                xs = x[:m].cpu().numpy()
                items = np.empty((m, n), dtype=oracle.ITEM)
                items["key"] = xs.view(np.uint64) ^ np.uint64(1 << 63)
                items["ref"] = 0
                res["cells"][f"rss_n{n}_{dname}"]["cpu_baseline"] = cpu_block(
                    items, RSS332_SPEC, m, 2 * m * n * 8, f"first {m} rows", kind="rss")
        del ins, ot
        torch.cuda.empty_cache()
    cells = res["cells"]
    for n in [int(x) for x in args.cfg3_ns.split(",")]:
        r = [v["ms_median"] for k, v in cells.items() if k.startswith(f"rss_n{n}_")]
        mg = [v["ms_median"] for k, v in cells.items() if k.startswith(f"merge_n{n}_")]
        res[f"n{n}_rss_over_merge_speed"] = round(float(np.mean(mg) / np.mean(r)), 3)
    res["min_frac_rss"] = min(v["frac"] for k, v in cells.items() if k.startswith("rss_n"))
    return res


def cfg4_inputs(torch, dev, lib, _lib, nseg):
    """Device-generated cfg4: lengths by inverse CDF of splitmix uniforms
    (oracle.geometric_lengths' recipe), f32 weights (u >> 40) * 2^-24, u32
    ids u & (2^26 - 1)."""
    sh = _lib.current_stream_handle(dev)
    u = torch.empty(nseg, dtype=torch.int64, device=dev)
    _lib.check(lib.nsg_fill_splitmix(u.data_ptr(), nseg, 8, 4, 0, sh))
    uf = ((u >> 11) & ((1 << 53) - 1)).to(torch.float64) * (1.0 / 2**53)
    q = 1.0 - 0.18
    k = torch.floor(torch.log1p(-uf * (1.0 - q**16)) / np.log(q)).to(torch.int64).clamp_(0, 15)
    lengths = 1 + k
    del u, uf, k
    off = torch.zeros(nseg + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lengths, 0, out=off[1:])
    e = int(off[-1].item())
    off32 = off.to(torch.int32)
    del off, lengths
    x = torch.empty(e, dtype=torch.int64, device=dev)
    _lib.check(lib.nsg_fill_splitmix(x.data_ptr(), e, 8, 40, 0, sh))
    w = ((x >> 40) & ((1 << 24) - 1)).to(torch.float32) * (2.0 ** -24)
    ids = (x & ((1 << 26) - 1)).to(torch.int32)
    del x
    return off32, w, ids, e


def wl_cfg4(args, torch, dev, grp, peak, want_cpu):
    import oracle
    from paper_2002_05599_b200 import _lib, batch
    from paper_2002_05599_b200.errors import CorrectnessFailure
    lib = _lib.lib()
    nseg = 67_108_864
    off, w, ids, e = cfg4_inputs(torch, dev, lib, _lib, nseg)
    wo, io = torch.empty_like(w), torch.empty_like(ids)
    ws = torch.empty(int(lib.nsg_segments_ws_bytes(nseg, e)), dtype=torch.uint8, device=dev)
    fn = lambda: batch.sort_segments(off, w, ids, descending=True, tie="unique", out_keys=wo,  # noqa: E731
                                     out_payload=io, workspace=ws, check=False)
    med, best = ev_time(torch, fn, args.reps)
    batch.sort_segments(off, w, ids, descending=True, tie="unique", out_keys=wo, out_payload=io, workspace=ws)
    bad = batch.verify_segments(off, w, wo, ids, io, descending=True, tie="unique")
    offh = off.cpu().numpy().view(np.uint32)
    lo, hi = 2_000_000, 2_040_000
    a, b = int(offh[lo]), int(offh[hi])
    sub = (offh[lo:hi + 1] - offh[lo]).astype(np.uint32)
    wh, ih = w[a:b].cpu().numpy(), ids[a:b].cpu().numpy().view(np.uint32)
    ek, ep = oracle.typed_sort_segments(sub, wh, ih, descending=True)
    if bad or not np.array_equal(wo[a:b].cpu().numpy(), ek) or \
            not np.array_equal(io[a:b].cpu().numpy().view(np.uint32), ep):
        raise CorrectnessFailure(f"cfg4 verification failed ({bad} bad segments)")
    blk = rate_block(2 * e * 8, nseg, e, med, best, peak)
    blk.update({"workload": "cfg4: 67,108,864 CSR segments, lengths truncated geometric 1..16 (p=0.18), "
                            "f32 weights desc + u32 ids (lexicographic)",
                "elements": e, "offsets_bytes_not_counted": 4 * (nseg + 1),
                "verified": "oracle on 40,000 segments + device order/multiset check of every segment"})
    if want_cpu:
        # reference recipe: bin by length (excluded), ns_run_sorter per bin
        m = 1 << 20
        lens = np.diff(offh[: m + 1].astype(np.int64))
        wk = w[: int(offh[m])].cpu().numpy()
        ik = ids[: int(offh[m])].cpu().numpy().view(np.uint32)
        okey = (((~oracle.to_ord(wk)) & np.uint64(0xFFFFFFFF)) << np.uint64(32)) | \
            ((~ik.astype(np.uint64)) & np.uint64(0xFFFFFFFF))
        bins = []
        for L in range(2, 17):
            sel = np.nonzero(lens == L)[0]
            if not len(sel):
                continue
            idx = (offh[sel][:, None].astype(np.int64) + np.arange(L)[None, :])
            it = np.empty((len(sel), L), dtype=oracle.ITEM)
            it["key"] = okey[idx]
            it["ref"] = ik[idx]
            bins.append(it)
        threads = oracle.cpu_count()
        t0 = time.perf_counter()
        kind = None
        for it in bins:
            kind = _cpu_run(it, _net_spec("best"), threads)
        dt = time.perf_counter() - t0
        blk["cpu_baseline"] = {"segments_per_s": m / dt, "elements_per_s": int(offh[m]) / dt,
                               "gbs": 2 * int(offh[m]) * 8 / dt / 1e9, "cores": threads, "kind": kind,
                               "sample": f"first {m} segments, binned by length (binning not timed), "
                                         "reference ns_run_sorter per bin on packed (~ord(w), ~id) keys"}
    del off, w, ids, wo, io, ws
    return blk


def wl_cfg5(args, torch, dev, grp, peak, want_cpu):
    """2^28 x 16 u64 key + u64 global index, split across the ranks by
    contiguous array ranges (shard.shard_rows); no collective on the data."""
    import oracle
    from paper_2002_05599_b200 import _lib, batch, shard
    from paper_2002_05599_b200.errors import CorrectnessFailure
    lib = _lib.lib()
    total = args.cfg5_rows
    lo, hi = shard.shard_rows(total, grp.rank, grp.world)
    rows = hi - lo
    sh = _lib.current_stream_handle(dev)
    kt = torch.empty(rows * 16, dtype=torch.int64, device=dev)
    _lib.check(lib.nsg_fill_splitmix(kt.data_ptr(), rows * 16, 8, 5, lo * 16, sh))
    kt = kt.view(torch.uint64).view(rows, 16)
    pt = torch.arange(lo * 16, hi * 16, dtype=torch.int64, device=dev).view(torch.uint64).view(rows, 16)
    ko, po = torch.empty_like(kt), torch.empty_like(pt)
    fn = lambda: batch.sort_rows(kt, pt, out_keys=ko, out_payload=po)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize(dev)
    times = []
    for _ in range(max(3, args.reps // 2)):
        grp.barrier()
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    my_ms = float(np.median(times))
    all_ms = grp.gather(my_ms)
    max_ms = max(all_ms)
    # verification: every row on device, oracle on a prefix of the shard
    from paper_2002_05599_b200 import registry
    bad = device_bad_rows(lib, _lib, registry, kt.view(torch.uint8), pt.view(torch.uint8), ko.view(torch.uint8),
                          po.view(torch.uint8), rows, 16, "uint64", "uint64", dev=dev)
    m = min(rows, 4096)
    ek, ep = oracle.typed_sort_rows(kt[:m].cpu().numpy(), pt[:m].cpu().numpy())
    if bad or not np.array_equal(ko[:m].cpu().numpy(), ek) or not np.array_equal(po[:m].cpu().numpy(), ep):
        raise CorrectnessFailure(f"cfg5 verification failed ({bad} bad rows)")
    if args.dump_dir:
        d = Path(args.dump_dir)
        d.mkdir(parents=True, exist_ok=True)
        np.save(d / f"cfg5_rank{grp.rank}.npy", np.stack([ko.cpu().numpy().reshape(-1), po.cpu().numpy().reshape(-1)]))
        (d / f"cfg5_rank{grp.rank}.json").write_text(json.dumps({"lo": lo, "hi": hi}))
    per_gpu_bytes = 2 * rows * 16 * 16
    tot_bytes = 2 * total * 16 * 16
    agg = tot_bytes / (max_ms / 1e3) / 1e9
    blk = {"workload": f"cfg5: {total} x n=16 uint64 key + uint64 global index, best_16 UNIQUE, "
                       f"split over {grp.world} GPU(s) by contiguous array ranges",
           "scaling": "strong", "arrays_total": total, "arrays_per_gpu": rows,
           "ms_max_over_ranks": round(max_ms, 4), "arrays_per_s": total / (max_ms / 1e3),
           "elements_per_s": total * 16 / (max_ms / 1e3), "gbs_aggregate": round(agg, 1),
           "frac_aggregate": round(agg / (peak * grp.world), 4),
           "gbs_per_gpu": [round(2 * (shard.shard_rows(total, r, grp.world)[1] - shard.shard_rows(total, r, grp.world)[0])
                                 * 256 / (t / 1e3) / 1e9, 1) for r, t in enumerate(all_ms)],
           "kernel": "net_sort n=16 best u64 p64 SoA UNIQUE",
           "verified": "device order/multiset check of every row + oracle on 4096 rows per shard"}
    del per_gpu_bytes
    if want_cpu:
        mm = 1 << 18
        items = np.empty((mm, 16), dtype=oracle.ITEM)
        items["key"] = kt[:mm].cpu().numpy()
        items["ref"] = pt[:mm].cpu().numpy()
        blk["cpu_baseline"] = cpu_block(items, _net_spec("best"), mm, 2 * mm * 16 * 16,
                                        f"first {mm} arrays", kind="network")
    del kt, pt, ko, po
    return blk


if __name__ == "__main__":
    main()
