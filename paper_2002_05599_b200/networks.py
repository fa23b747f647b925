"""Comparator networks for n = 2..16: the data the CUDA generator compiles.

Mirrors the reference's network layer (`pkg/src/netsort/networks.py`):

* Bose-Nelson construction (reference networks.py:88-122, `generate_bose_nelson`)
  re-derived here from the published recursion (Bose & Nelson 1962): sort the
  two halves, then merge them with the recursive split merge.
* "Best" tables (reference `data/networks/best_NN.txt`, provenance
  `tools/make_network_tables.py:3-14,56-80`): n <= 8 is the Bose-Nelson list,
  n = 10 is the classic 29-comparator / depth-9 network, n = 16 is Green's
  60-comparator / depth-10 network, n = 9 and n = 11..15 are top-channel
  restrictions (reference networks.py:265-274).
* Families best / bn-l / bn-p / bn-r (reference networks.py:277-292).  BN-L,
  BN-P and BN-R are three schedules of ONE comparator DAG (BN-P keeps per-channel
  order, BN-R flattens to the locality order), so they produce bit-identical
  outputs and the device code compiles a single BN DAG for all three.

`tests/test_networks.py` pins every list here against the reference's own
`family_network` output (tests/golden/networks.json).
"""

from __future__ import annotations

import functools
from dataclasses import dataclass
from typing import NamedTuple

from .errors import TooLargeForExhaustive, UnsupportedSize

FAMILY_KEYS = ("best", "bn-l", "bn-p", "bn-r")
FAMILY_LABELS = {"best": "Best", "bn-l": "BN-L", "bn-p": "BN-P", "bn-r": "BN-R"}
LABEL_TO_FAMILY = {v: k for k, v in FAMILY_LABELS.items()}
BEST_KNOWN = "BestKnown"
BN_LOCALITY = "BN-Locality"
BN_PARALLEL = "BN-Parallel"
BN_RECURSIVE = "BN-Recursive"
FAMILY_TAGS = {"best": BEST_KNOWN, "bn-l": BN_LOCALITY, "bn-p": BN_PARALLEL,
               "bn-r": BN_RECURSIVE}

MIN_UNROLLED = 2
MAX_UNROLLED = 16
MAX_EXHAUSTIVE = 24

# Device DAG ids: the CUDA kernels are compiled once per DAG, not per family.
DAG_BEST = 0
DAG_BN = 1


def family_dag(family: str) -> int:
    if family not in FAMILY_KEYS:
        raise ValueError(f"unknown family {family!r}")
    return DAG_BEST if family == "best" else DAG_BN


class Comparator(NamedTuple):
    low: int
    high: int


@dataclass(frozen=True)
class Network:
    n: int
    comparators: tuple
    ordering_tag: str = BEST_KNOWN

    def __post_init__(self):
        for lo, hi in self.comparators:
            if not 0 <= lo < hi < self.n:
                raise ValueError(f"comparator ({lo},{hi}) invalid for {self.n} channels")

    @property
    def size(self) -> int:
        return len(self.comparators)


# ---------------------------------------------------------------------------
# Bose-Nelson
# ---------------------------------------------------------------------------

def _bn_merge(a: int, na: int, b: int, nb: int, out: list) -> None:
    """Merge sorted runs a[0:na] and b[0:nb] (Bose-Nelson merge recursion)."""
    if na == 1 and nb == 1:
        out.append(Comparator(a, b))
        return
    if na == 1 and nb == 2:
        out += [Comparator(a, b + 1), Comparator(a, b)]
        return
    if na == 2 and nb == 1:
        out += [Comparator(a, b), Comparator(a + 1, b)]
        return
    ha = na // 2
    hb = (nb + 1) // 2 if na % 2 == 0 else nb // 2
    _bn_merge(a, ha, b, hb, out)
    _bn_merge(a + ha, na - ha, b + hb, nb - hb, out)
    _bn_merge(a + ha, na - ha, b, hb, out)


def _bn_sort(base: int, m: int, out: list) -> None:
    if m < 2:
        return
    h = m // 2
    _bn_sort(base, h, out)
    _bn_sort(base + h, m - h, out)
    _bn_merge(base, h, base + h, m - h, out)


def generate_bose_nelson(n: int) -> Network:
    """Bose-Nelson network in recursion (locality) order."""
    if n < 0:
        raise ValueError("channel count must be nonnegative")
    out: list = []
    _bn_sort(0, n, out)
    return Network(n, tuple(out), BN_LOCALITY)


def bose_nelson_merger(n: int) -> tuple:
    out: list = []
    if n >= 2:
        _bn_merge(0, n // 2, n // 2, n - n // 2, out)
    return tuple(out)


# ---------------------------------------------------------------------------
# Best-known tables (0-based, one inner list per parallel level)
# ---------------------------------------------------------------------------

# Classic 29-comparator sorter on 10 channels, depth 9.
_BEST10_LEVELS = (
    ((4, 9), (3, 8), (2, 7), (1, 6), (0, 5)),
    ((1, 4), (6, 9), (0, 3), (5, 8)),
    ((0, 2), (3, 6), (7, 9)),
    ((0, 1), (2, 4), (5, 7), (8, 9)),
    ((1, 2), (4, 6), (7, 8), (3, 5)),
    ((2, 5), (6, 8), (1, 3), (4, 7)),
    ((2, 3), (6, 7)),
    ((3, 4), (5, 6)),
    ((4, 5),),
)

# Green's 60-comparator sorter on 16 channels, depth 10.
_BEST16_LEVELS = (
    ((0, 1), (2, 3), (4, 5), (6, 7), (8, 9), (10, 11), (12, 13), (14, 15)),
    ((0, 2), (4, 6), (8, 10), (12, 14), (1, 3), (5, 7), (9, 11), (13, 15)),
    ((0, 4), (8, 12), (1, 5), (9, 13), (2, 6), (10, 14), (3, 7), (11, 15)),
    ((0, 8), (1, 9), (2, 10), (3, 11), (4, 12), (5, 13), (6, 14), (7, 15)),
    ((5, 10), (6, 9), (3, 12), (13, 14), (7, 11), (1, 2), (4, 8)),
    ((1, 4), (7, 13), (2, 8), (11, 14)),
    ((2, 4), (5, 6), (9, 10), (11, 13), (3, 8), (7, 12)),
    ((6, 8), (10, 12), (3, 5), (7, 9)),
    ((3, 4), (5, 6), (7, 8), (9, 10), (11, 12)),
    ((6, 7), (8, 9)),
)


def _flatten(levels) -> tuple:
    return tuple(Comparator(a, b) for level in levels for a, b in level)


def restrict_top_channel(net: Network) -> Network:
    """Drop channel n-1 and every comparator touching it (pin it to +inf)."""
    top = net.n - 1
    kept = tuple(c for c in net.comparators if top not in c)
    return Network(net.n - 1, kept, net.ordering_tag)


@functools.lru_cache(maxsize=None)
def best_network(n: int) -> Network:
    if not MIN_UNROLLED <= n <= MAX_UNROLLED:
        raise UnsupportedSize(f"no embedded best-known network for n={n}")
    if n <= 8:
        return Network(n, generate_bose_nelson(n).comparators, BEST_KNOWN)
    if n <= 10:
        net = Network(10, _flatten(_BEST10_LEVELS), BEST_KNOWN)
    else:
        net = Network(16, _flatten(_BEST16_LEVELS), BEST_KNOWN)
    while net.n > n:
        net = restrict_top_channel(net)
    return net


@functools.lru_cache(maxsize=None)
def family_network(family: str, n: int) -> Network:
    if family not in FAMILY_KEYS:
        raise ValueError(f"unknown family {family!r}")
    if not MIN_UNROLLED <= n <= MAX_UNROLLED:
        raise UnsupportedSize(f"family {family} supports n in 2..16, got {n}")
    if family == "best":
        return best_network(n)
    bn = generate_bose_nelson(n)
    if family == "bn-l":
        return bn
    if family == "bn-p":
        return reorder_parallelism(bn)
    return Network(n, bn.comparators, BN_RECURSIVE)


# ---------------------------------------------------------------------------
# Levels / verification
# ---------------------------------------------------------------------------

def compute_levels(net: Network) -> tuple:
    """Greedy earliest-level schedule; same-channel order is preserved."""
    ready = [0] * max(net.n, 1)
    levels: list = []
    for c in net.comparators:
        lvl = max(ready[c.low], ready[c.high])
        if lvl == len(levels):
            levels.append([])
        levels[lvl].append(c)
        ready[c.low] = ready[c.high] = lvl + 1
    return tuple(tuple(level) for level in levels)


def depth(net: Network) -> int:
    return len(compute_levels(net))


def reorder_parallelism(net: Network) -> Network:
    flat = tuple(c for level in compute_levels(net) for c in level)
    return Network(net.n, flat, BN_PARALLEL)


def verify_zero_one(net: Network) -> bool:
    """0/1 principle over all 2^n inputs, bit-sliced into Python ints."""
    n = net.n
    if n > MAX_EXHAUSTIVE:
        raise TooLargeForExhaustive(f"n={n} exceeds {MAX_EXHAUSTIVE}")
    if n < 2:
        return True
    total = 1 << n
    chans = []
    for i in range(n):
        # bit v of channel i = bit i of input vector v
        block = (1 << (1 << i)) - 1           # 2^i ones
        period = block << (1 << i)            # pattern of one period
        word, width = period, 1 << (i + 1)
        while width < total:                  # double the period up to 2^n bits
            word |= word << width
            width <<= 1
        chans.append(word)
    for lo, hi in net.comparators:
        a, b = chans[lo], chans[hi]
        chans[lo], chans[hi] = a & b, a | b
    full = (1 << total) - 1
    return all(chans[i] & (chans[i + 1] ^ full) == 0 for i in range(n - 1))


def dag_comparators(dag: int, n: int) -> tuple:
    """Comparator list the device compiles for (dag, n), level-scheduled."""
    if dag == DAG_MERGE:
        net = merge_network(n)
    else:
        net = best_network(n) if dag == DAG_BEST else generate_bose_nelson(n)
    return tuple(c for level in compute_levels(net) for c in level)


# ---------------------------------------------------------------------------
# Merge networks for 32 / 64 items (the device's thread-per-array "merge"
# sorter; no counterpart in the reference, which switches to RSS above 16)
# ---------------------------------------------------------------------------

DAG_MERGE = 2


def _odd_even_merge(lo: int, n: int, r: int, out: list) -> None:
    """Batcher's odd-even merge of the two sorted halves of a[lo:lo+n] (stride r)."""
    step = 2 * r
    if step < n:
        _odd_even_merge(lo, n, step, out)
        _odd_even_merge(lo + r, n, step, out)
        for i in range(lo + r, lo + n - r, step):
            out.append(Comparator(i, i + r))
    else:
        out.append(Comparator(lo, lo + r))


@functools.lru_cache(maxsize=None)
def merge_network(n: int) -> Network:
    """n = 32 / 64: two sorted halves (Green-16 at the bottom) + odd-even merge.

    32 items: 2 x 60 + 65 = 185 comparators (the best known size), depth 15.
    """
    if n == 16:
        return best_network(16)
    if n not in (32, 64):
        raise UnsupportedSize(f"merge networks are built for 32 and 64 items, got {n}")
    half = merge_network(n // 2)
    comps = list(half.comparators)
    comps += [Comparator(a + n // 2, b + n // 2) for a, b in half.comparators]
    _odd_even_merge(0, n, 1, comps)
    return Network(n, tuple(comps), "OddEvenMerge")
