"""The device lane: same surface as the reference's lane modules.

Reference: `backend.py:37-53` re-exports either `_native` (Cython over the C
core) or `_pybackend`.  This package has exactly one lane, LANE = "cuda",
backed by libnsg.so; there is no CPU fallback (a missing library or GPU
raises).  Functions keep the reference's names, arguments and error behaviour:

  run_sorter(spec, arr, n=None)        _native.pyx:171-187
  run_sorter_many(spec, rows)          _native.pyx:190-208   <- the hot path
  swap_pairs(code, rows)               _native.pyx:211-220
  classify_block_u64(keys, s0,s1,s2,b) _native.pyx:223-235
  lcg_next / fill_items / fingerprint / check_sorted   (host utilities)

`rows` may be a numpy `ITEM_DTYPE` array (host buffers; copies are pipelined
with the sort inside the library) or a CUDA tensor of shape (m, n, 2) and
dtype int64/uint64 holding the same packed items (device-resident, in place,
stream-ordered on torch's current stream).
"""

from __future__ import annotations

import numpy as np

from . import registry
from ._lib import check, current_stream_handle, lib, load_library, make_spec
from .errors import ConfigurationError, UnsupportedSize
from .items import ITEM_DTYPE

LANE = "cuda"
TIMER_KIND = "nanos"
FP_PRIME = (1 << 61) - 1
LCG_MULTIPLIER = 48271
LCG_MODULUS = 2147483647


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _check_items(arr, need: int) -> None:
    # reference item_ptr (_native.pyx:85-95)
    if not isinstance(arr, np.ndarray) or arr.dtype != ITEM_DTYPE:
        raise ConfigurationError("expected a structured item array")
    if not arr.flags.c_contiguous:
        raise ConfigurationError("item array must be C-contiguous")
    if arr.size < need:
        raise ConfigurationError(f"array holds {arr.size} items, need {need}")


def _check_item_tensor(t) -> tuple:
    import torch
    if not t.is_cuda or t.dtype not in (torch.int64, torch.uint64) or t.dim() != 3 or t.shape[2] != 2:
        raise ConfigurationError("expected a CUDA (m, n, 2) int64/uint64 tensor of packed items")
    if not t.is_contiguous():
        raise ConfigurationError("item tensor must be contiguous")
    return int(t.shape[0]), int(t.shape[1])


def run_sorter_many(spec, rows) -> None:
    """Sort every row of `rows` in place with `spec` (kind network / RSS / IS)."""
    l = lib()
    sp = make_spec(spec)
    network = spec[0] == registry.KIND_NETWORK
    if _is_torch(rows):
        m, n = _check_item_tensor(rows)
        rc = l.nsg_run_sorter_many(sp, rows.data_ptr(), m, n, current_stream_handle(rows.device))
        check(rc, network=network)
        return
    if not isinstance(rows, np.ndarray) or rows.ndim != 2:
        raise ConfigurationError("expected a 2-D array of input rows")
    m, n = rows.shape
    _check_items(rows, m * n)
    check(l.nsg_run_sorter_many_host(sp, rows.ctypes.data, m, n), network=network)


def run_sorter(spec, arr, n=None) -> None:
    """Sort the first n items of one item array in place (`_native.pyx:171-187`)."""
    nn = len(arr) if n is None else int(n)
    if spec[0] == registry.KIND_NETWORK and nn >= 2 and not 2 <= nn <= 16:
        raise UnsupportedSize(f"network sorters cover 2..16 items, got {nn}")
    _check_items(arr, nn)
    if nn < 2:
        return
    view = arr[:nn].reshape(1, nn)
    run_sorter_many(spec, view)


def swap_pairs(code: int, rows) -> None:
    """One conditional swap per (left, right) item pair, in place."""
    l = lib()
    if _is_torch(rows):
        m, two = _check_item_tensor(rows)
        if two != 2:
            raise ConfigurationError("expected an (m, 2) array of item pairs")
        check(l.nsg_swap_pairs(int(code), rows.data_ptr(), m, current_stream_handle(rows.device)))
        return
    if rows.ndim != 2 or rows.shape[1] != 2:
        raise ConfigurationError("expected an (m, 2) array of item pairs")
    _check_items(rows, rows.shape[0] * 2)
    import torch
    d = torch.from_numpy(rows.view(np.uint64).reshape(-1, 2, 2)).cuda()
    check(l.nsg_swap_pairs(int(code), d.data_ptr(), rows.shape[0], current_stream_handle()))
    rows.view(np.uint64).reshape(-1, 2, 2)[...] = d.cpu().numpy()


def classify_block_u64(keys, s0, s1, s2, block=1) -> np.ndarray:
    """Bucket tags 0..3 for u64 keys (`ns_classify_block`)."""
    import torch
    if not 1 <= int(block) <= 5:
        raise ConfigurationError("block size must be in 1..5")
    l = lib()
    host = not _is_torch(keys)
    kt = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64)).cuda() if host else keys.contiguous()
    n = kt.numel()
    tags = torch.empty(n, dtype=torch.uint8, device=kt.device)
    if n:
        check(l.nsg_classify_block(kt.data_ptr(), n, int(s0), int(s1), int(s2), int(block),
                                   tags.data_ptr(), current_stream_handle(kt.device)))
    return tags.cpu().numpy() if host else tags


# ---------------------------------------------------------------------------
# host utilities (reference netsort_core.c:38-100)
# ---------------------------------------------------------------------------

def lcg_next(seed: int) -> int:
    return int(load_library().nsg_lcg_next(int(seed) & 0xFFFFFFFF))


def lcg_stream(seed: int, count: int) -> np.ndarray:
    """[lcg^1(seed), ..., lcg^count(seed)] by jump-ahead doubling (vectorised)."""
    out = np.empty(count, dtype=np.uint64)
    if count == 0:
        return out
    out[0] = (int(seed) * LCG_MULTIPLIER) % LCG_MODULUS
    have, mult = 1, LCG_MULTIPLIER
    while have < count:
        take = min(have, count - have)
        mult_k = pow(LCG_MULTIPLIER, have, LCG_MODULUS)
        out[have:have + take] = (out[:take] * np.uint64(mult_k)) % np.uint64(LCG_MODULUS)
        have += take
    return out


def fill_items(arr: np.ndarray, seed: int) -> int:
    """ns_fill: key_i, ref_i from consecutive LCG draws; returns the final state."""
    n = len(arr)
    s = lcg_stream(seed, 2 * n)
    arr["key"] = s[0::2]
    arr["ref"] = s[1::2]
    return int(s[-1]) if n else int(seed)


def _fp_once(keys, z: int, p: int) -> int:
    v = 1
    for k in keys:
        v = (v * ((z - k) % p)) % p
    return v


def fingerprint(arr, n=None, z=1, p=FP_PRIME) -> tuple:
    """Multiset fingerprint prod(z - key) mod p with the z-bump search."""
    n = len(arr) if n is None else n
    keys = [int(k) for k in arr["key"][:n]]
    while True:
        v = _fp_once(keys, z % p, p)
        if v != 0:
            return v, z
        z += 1


def check_sorted(arr, n=None) -> bool:
    n = len(arr) if n is None else n
    k = arr["key"][:n]
    return bool(np.all(k[:-1] <= k[1:])) if n > 1 else True


def hybrid_stats(spec, arr):
    raise ConfigurationError("hybrid quicksort is a single-array CPU sorter: out of scope of the device lane")


def measure_one_array_repeat(spec, size, iterations, seed):
    raise ConfigurationError("OneArrayRepeat is a CPU cycle-count harness: use bench.py on the device lane")


def measure_array_in_row(spec, size, narrays, seed):
    raise ConfigurationError("ArrayInRow is a CPU cycle-count harness: use bench.py on the device lane")
