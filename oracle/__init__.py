"""CPU oracle for the device sorter -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this package, as the checker or the timed CPU
baseline.  The product (paper_2002_05599_b200) never imports it.

Two CPU implementations live here:
  * liboracle.so          -- our C restatement of the reference hot path
                             (netsort_oracle.c, every function cites its
                             reference file:line);
  * _ref/libnetsort_ref.so -- the reference's OWN C core compiled from its
                             sources (oracle/Makefile), driven by ref_driver.c.
Parity is pinned: tests/test_oracle.py checks the restatement against the
golden vectors produced by the reference (tests/golden/make_golden.py) and,
where _ref is built, against the reference binary itself.

Adapters map the BASELINE configs' typed SoA batches to the
reference's (u64 key, u64 ref) items and back: u32 zero-extended; i32/i64 sign
flip; f32/f64 orderable bits; descending = complemented key (and payload in
UNIQUE mode); payload -> ref.
"""

from __future__ import annotations

import ctypes
import json
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
GOLDEN = ROOT / "tests" / "golden"
ITEM = np.dtype([("key", "<u8"), ("ref", "<u8")])
FAMILIES = ("best", "bn-l", "bn-p", "bn-r")


class OrNets(ctypes.Structure):
    _fields_ = [("pairs", ctypes.c_void_p), ("off", ctypes.c_void_p)]


class OrSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("base_kind", ctypes.c_int), ("oversampling", ctypes.c_int),
                ("threshold", ctypes.c_int), ("seed", ctypes.c_uint32), ("unique", ctypes.c_int)]


class NsSpec(ctypes.Structure):  # the reference's ns_spec, netsort_core.h:156-171
    _fields_ = [(f, ctypes.c_int) for f in ("kind", "family", "swap", "ins_variant", "base_kind",
                                             "rss_oversampling", "rss_block", "rss_threshold")] + \
               [("rss_sample_seed", ctypes.c_uint32)] + \
               [(f, ctypes.c_int) for f in ("qs_base_is_rss", "qs_threshold", "qs_depth_factor",
                                             "qs_final_pass", "pivot_swap")]


_lib = None
_ref = None
_tables: dict = {}


def build() -> None:
    """Compile liboracle.so (+ _ref when the reference sources are present)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)


def lib():
    global _lib
    if _lib is None:
        path = HERE / "liboracle.so"
        if not path.exists():
            build()
        l = ctypes.CDLL(str(path))
        l.or_lcg_next.restype = ctypes.c_uint32
        l.or_lcg_next.argtypes = [ctypes.c_uint32]
        l.or_run_many.restype = ctypes.c_int
        l.or_run_many.argtypes = [ctypes.POINTER(OrSpec), ctypes.POINTER(OrNets), ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_long, ctypes.c_int]
        l.or_classify.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_void_p]
        l.or_sort_segments.argtypes = [ctypes.POINTER(OrNets), ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_int]
        _lib = l
    return _lib


def ref_lib():
    """The reference's own C core (None when it was not built)."""
    global _ref
    if _ref is None:
        path = HERE / "_ref" / "libnetsort_ref.so"
        if not path.exists():
            return None
        l = ctypes.CDLL(str(path))
        l.ref_run_many.restype = ctypes.c_int
        l.ref_run_many.argtypes = [ctypes.POINTER(NsSpec), ctypes.c_void_p, ctypes.c_int64, ctypes.c_long,
                                   ctypes.c_int]
        _ref = l
    return _ref


def nets(family: str):
    """Comparator tables of a family, from the reference-generated golden."""
    if family not in _tables:
        doc = json.loads((GOLDEN / "networks.json").read_text())["families"][family]
        pairs, off = [], [0, 0, 0]
        for n in range(2, 17):
            pairs += [x for c in doc[str(n)] for x in c]
            off.append(len(pairs) // 2)
        pa = np.array(pairs, dtype=np.uint8)
        oa = np.array(off, dtype=np.int32)  # off[n] .. off[n+1]
        _tables[family] = (pa, oa, OrNets(pa.ctypes.data, oa.ctypes.data))
    return _tables[family][2]


def lcg_next(s: int) -> int:
    return int(lib().or_lcg_next(s & 0xFFFFFFFF))


def fill_items(arr: np.ndarray, seed: int) -> int:
    """ns_fill (netsort_core.c:42-50), sequentially: key_i, ref_i are the
    (2i+1)-th and (2i+2)-th draws; returns the final state."""
    s = int(seed) & 0xFFFFFFFF
    keys = np.empty(len(arr), dtype=np.uint64)
    refs = np.empty(len(arr), dtype=np.uint64)
    for i in range(len(arr)):
        s = lcg_next(s)
        keys[i] = s
        s = lcg_next(s)
        refs[i] = s
    arr["key"], arr["ref"] = keys, refs
    return s


def lcg_jump(seed: int, k: int) -> int:
    """The state after k draws: seed * 48271^k mod (2^31 - 1) (k >= 1)."""
    return (int(seed) * pow(48271, int(k), 2147483647)) % 2147483647 if k else int(seed)


FP_PRIME = (1 << 61) - 1


def fingerprint(keys, z: int = 1) -> tuple:
    """ns_fp_at / ns_fp_search (netsort_core.c:70-91) over python ints."""
    keys = [int(k) % FP_PRIME for k in keys]
    z = int(z)
    while True:
        zz, v = z % FP_PRIME, 1
        for k in keys:
            v = v * ((zz - k) % FP_PRIME) % FP_PRIME
        if v:
            return v, z
        z += 1


def _spec(kind: int, rss_cfg: str = "332", base: str = "net", threshold: int = 16, seed: int = 0x5EED,
          unique: bool = False) -> OrSpec:
    return OrSpec(kind, 0 if base == "net" else 1, int(rss_cfg[1]), threshold, seed, int(unique))


def run_items(items: np.ndarray, *, kind: str = "network", family: str = "best", rss_cfg: str = "332",
              base: str = "net", unique: bool = False, threads: int = 1, threshold: int = 16,
              seed: int = 0x5EED) -> np.ndarray:
    """Sort each row of an (m, n) ITEM array in place with the restatement."""
    assert items.dtype == ITEM and items.ndim == 2 and items.flags.c_contiguous
    k = {"network": 0, "insertion": 1, "rss": 2}[kind]
    sp = _spec(k, rss_cfg, base, threshold, seed, unique)
    rc = lib().or_run_many(ctypes.byref(sp), ctypes.byref(nets(family)), items.ctypes.data,
                           items.shape[0], items.shape[1], threads)
    if rc != 0:
        raise ValueError(f"oracle rejected the spec (status {rc})")
    return items


def ref_run_items(items: np.ndarray, spec_tuple, threads: int = 1) -> np.ndarray:
    """Sort with the reference's OWN compiled core (ns_run_sorter)."""
    l = ref_lib()
    if l is None:
        raise RuntimeError("oracle/_ref/libnetsort_ref.so not built")
    vals = [int(x) for x in tuple(spec_tuple)]
    sp = NsSpec(*vals)
    rc = l.ref_run_many(ctypes.byref(sp), items.ctypes.data, items.shape[0], items.shape[1], threads)
    if rc != 0:
        raise ValueError(f"reference rejected the spec (status {rc})")
    return items


def classify(keys: np.ndarray, s0: int, s1: int, s2: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    tags = np.empty(len(keys), dtype=np.uint8)
    lib().or_classify(keys.ctypes.data, len(keys), s0, s1, s2, tags.ctypes.data)
    return tags


def sort_segments_items(offsets: np.ndarray, items: np.ndarray, family: str = "best", unique: bool = True):
    off = np.ascontiguousarray(offsets, dtype=np.uint32)
    lib().or_sort_segments(ctypes.byref(nets(family)), off.ctypes.data, len(off) - 1, items.ctypes.data,
                           int(unique))
    return items


# ---------------------------------------------------------------------------
# Adapters
# ---------------------------------------------------------------------------

def to_ord(keys: np.ndarray, descending: bool = False) -> np.ndarray:
    """Typed keys -> order-preserving unsigned integers (u64)."""
    k = np.asarray(keys)
    if k.dtype == np.uint32 or k.dtype == np.uint64:
        o = k.astype(np.uint64)
        bits = k.dtype.itemsize * 8
    elif k.dtype == np.int32 or k.dtype == np.int64:
        bits = k.dtype.itemsize * 8
        u = k.view(np.uint32 if bits == 32 else np.uint64).astype(np.uint64)
        o = u ^ np.uint64(1 << (bits - 1))
    elif k.dtype == np.float32 or k.dtype == np.float64:
        bits = k.dtype.itemsize * 8
        u = k.view(np.uint32 if bits == 32 else np.uint64).astype(np.uint64)
        sign = np.uint64(1 << (bits - 1))
        mask = np.uint64((1 << bits) - 1)
        neg = (u & sign) != 0
        o = np.where(neg, (~u) & mask, u | sign)
    else:
        raise TypeError(k.dtype)
    if descending:
        o = (~o) & np.uint64((1 << bits) - 1)
    return o


def typed_sort_rows(keys: np.ndarray, payload=None, *, family: str = "best", descending: bool = False,
                    unique: bool = True, kind: str = "network", rss_cfg: str = "332", base: str = "net",
                    threads: int = 1):
    """Expected output of batch.sort_rows computed through the oracle."""
    keys = np.asarray(keys)
    m, n = keys.shape
    items = np.empty((m, n), dtype=ITEM)
    items["key"] = to_ord(keys, descending)
    # ref carries the original column index so keys and payload come back exactly
    col = np.broadcast_to(np.arange(n, dtype=np.uint64), (m, n))
    if payload is not None:
        p = np.asarray(payload)
        pu = p.view(np.uint32 if p.dtype.itemsize == 4 else np.uint64).astype(np.uint64)
        if unique and descending:
            pu = (~pu) & np.uint64((1 << (8 * p.dtype.itemsize)) - 1)
        if unique:
            # lexicographic (key, payload): payload in the high bits, index low
            # would overflow for u64 payloads; sort by (key, payload) directly
            items["ref"] = pu
        else:
            items["ref"] = pu
    else:
        items["ref"] = col
    if payload is not None and unique:
        run_items(items, kind=kind, family=family, rss_cfg=rss_cfg, base=base, unique=True, threads=threads)
    else:
        run_items(items, kind=kind, family=family, rss_cfg=rss_cfg, base=base, unique=False, threads=threads)
    # map back: recover original keys/payload by locating values
    out_keys = np.empty_like(keys)
    out_pay = None
    if payload is None:
        idx = items["ref"].astype(np.int64)
        out_keys[...] = np.take_along_axis(keys, idx, axis=1)
    else:
        out_keys[...] = from_ord(items["key"], keys.dtype, descending)
        pu = items["ref"]
        if unique and descending:
            pu = (~pu) & np.uint64((1 << (8 * p.dtype.itemsize)) - 1)
        out_pay = pu.astype(p.view(np.uint32 if p.dtype.itemsize == 4 else np.uint64).dtype).view(p.dtype)
    return out_keys, out_pay


def typed_sort_segments(offsets, keys, payload=None, *, family: str = "best", descending: bool = False,
                        unique: bool = True):
    """Expected output of batch.sort_segments (CSR) through the oracle."""
    keys = np.asarray(keys)
    items = np.empty(len(keys), dtype=ITEM)
    items["key"] = to_ord(keys, descending)
    if payload is None:
        items["ref"] = np.arange(len(keys), dtype=np.uint64)
        sort_segments_items(offsets, items, family=family, unique=False)
        return keys[items["ref"].astype(np.int64)], None
    p = np.asarray(payload)
    pbits = 8 * p.dtype.itemsize
    pu = p.view(np.uint32 if pbits == 32 else np.uint64).astype(np.uint64)
    if unique and descending:
        pu = (~pu) & np.uint64((1 << pbits) - 1)
    items["ref"] = pu
    sort_segments_items(offsets, items, family=family, unique=unique)
    out_k = from_ord(items["key"], keys.dtype, descending)
    pu = items["ref"]
    if unique and descending:
        pu = (~pu) & np.uint64((1 << pbits) - 1)
    return out_k, pu.astype(np.uint32 if pbits == 32 else np.uint64).view(p.dtype)


def geometric_lengths(nseg: int, seed: int, p: float = 0.18, lo: int = 1, hi: int = 16) -> np.ndarray:
    """cfg4 segment lengths: truncated geometric on lo..hi by inverse CDF of a
    counter-based uniform (splitmix64 >> 11 / 2^53)."""
    u = (splitmix(nseg, seed) >> np.uint64(11)).astype(np.float64) * (1.0 / 2**53)
    q = 1.0 - p
    span = hi - lo + 1
    # P(L <= lo + k) = (1 - q^(k+1)) / (1 - q^span)
    k = np.floor(np.log1p(-u * (1.0 - q**span)) / np.log(q)).astype(np.int64)
    return (lo + np.clip(k, 0, span - 1)).astype(np.uint32)


def from_ord(o: np.ndarray, dtype, descending: bool = False) -> np.ndarray:
    dtype = np.dtype(dtype)
    bits = dtype.itemsize * 8
    mask = np.uint64((1 << bits) - 1)
    o = np.asarray(o, dtype=np.uint64)
    if descending:
        o = (~o) & mask
    sign = np.uint64(1 << (bits - 1))
    if dtype.kind == "u":
        u = o
    elif dtype.kind == "i":
        u = o ^ sign
    else:
        pos = (o & sign) != 0
        u = np.where(pos, o ^ sign, (~o) & mask)
    ut = np.uint32 if bits == 32 else np.uint64
    return u.astype(ut).view(dtype)


# ---------------------------------------------------------------------------
# Seeded synthetic inputs (identical to nsg_fill_splitmix on the device)
# ---------------------------------------------------------------------------

def splitmix(count: int, seed: int, first: int = 0, elem_bytes: int = 8) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(first, first + count, dtype=np.uint64)
        x = np.uint64(seed) + i * np.uint64(0xD1B54A32D192ED03)
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    if elem_bytes == 8:
        return x
    return (x >> np.uint64(32)).astype(np.uint32)


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
