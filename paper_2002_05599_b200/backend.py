"""The device lane: same surface as the reference's lane modules.

Reference: `backend.py:37-53` re-exports either `_native` (Cython over the C
core) or `_pybackend`.  This package has exactly one lane, LANE = "cuda",
backed by libnsg.so; there is no CPU fallback (a missing library or GPU
raises).  Functions keep the reference's names, arguments and error behaviour:

  run_sorter(spec, arr, n=None)        _native.pyx:171-187
  run_sorter_many(spec, rows)          _native.pyx:190-208   <- the hot path
  swap_pairs(code, rows)               _native.pyx:211-220
  classify_block_u64(keys, s0,s1,s2,b) _native.pyx:223-235
  lcg_next / fill_items / fingerprint / check_sorted   netsort_core.c:38-100 (on the device)
  measure_array_in_row(spec, size, narrays, seed)      _native.pyx:285-308 (CUDA-event timed)

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
        import torch
        m, n = _check_item_tensor(rows)
        with torch.cuda.device(rows.device):
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
        import torch
        with torch.cuda.device(rows.device):
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
        with torch.cuda.device(kt.device):
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


def _items_on_device(arr, n=None):
    """(CUDA (n, 2) u64 tensor of items, host array to copy back or None).

    numpy ITEM_DTYPE arrays are staged to the device (the lane computes on the
    GPU only); CUDA tensors whose last dimension is 2 (packed items) are used
    in place."""
    import torch
    if _is_torch(arr):
        if not arr.is_cuda or arr.dtype not in (torch.int64, torch.uint64) or arr.shape[-1] != 2 \
                or not arr.is_contiguous():
            raise ConfigurationError("expected a contiguous CUDA (..., 2) int64/uint64 tensor of packed items")
        flat = arr.view(-1, 2)
        nn = flat.shape[0] if n is None else int(n)
        if nn > flat.shape[0]:
            raise ConfigurationError(f"array holds {flat.shape[0]} items, need {nn}")
        return flat[:nn], None
    nn = len(arr) if n is None else int(n)
    _check_items(arr, nn)
    host = arr[:nn].view(np.uint64).reshape(nn, 2)
    lib()
    return torch.from_numpy(host.view(np.int64)).cuda(), host


def fill_items(arr, seed: int) -> int:
    """ns_fill (netsort_core.c:42-50) on the device: key_i, ref_i from the
    (2i+1)-th and (2i+2)-th LCG draws; returns the final generator state."""
    import ctypes
    import torch
    l = lib()
    if _is_torch(arr):
        items, host = _items_on_device(arr)
    else:
        _check_items(arr, len(arr))
        host = arr.view(np.uint64).reshape(len(arr), 2)
        items = torch.empty((len(arr), 2), dtype=torch.int64, device="cuda")
    n = items.shape[0]
    final = ctypes.c_uint32(0)
    ptr = items.data_ptr() if n else None
    with torch.cuda.device(items.device):
        check(l.nsg_fill_lcg(ptr, 16, ptr + 8 if n else None, 16, n, int(seed) & 0xFFFFFFFF,
                             ctypes.byref(final), current_stream_handle(items.device)))
    if host is not None and n:
        host[...] = items.cpu().numpy().view(np.uint64)
    return int(final.value)


def _fp_device(items, z: int, ws, out) -> int:
    import torch
    l = lib()
    n = items.shape[0]
    with torch.cuda.device(items.device):
        check(l.nsg_fingerprint(items.data_ptr() if n else None, 8, 16, n, int(z) & 0xFFFFFFFFFFFFFFFF,
                                ws.data_ptr(), ws.numel(), out.data_ptr(), current_stream_handle(items.device)))
    return int(out.item()) & 0xFFFFFFFFFFFFFFFF


def fingerprint(arr, n=None, z=1, p=FP_PRIME) -> tuple:
    """ns_fp_search (netsort_core.c:81-91): the first z' >= z whose multiset
    fingerprint prod(z' - key) mod p is nonzero, and that value; computed on
    the device (nsg_fingerprint), the z bump on the host as in the reference."""
    import torch
    if p != FP_PRIME:
        raise ConfigurationError("the device lane fingerprints modulo FP_PRIME = 2^61 - 1 only")
    items, _ = _items_on_device(arr, n)
    ws = torch.empty(int(load_library().nsg_fingerprint_ws_bytes()), dtype=torch.uint8, device=items.device)
    out = torch.empty(1, dtype=torch.int64, device=items.device)
    z = int(z)
    while True:
        v = _fp_device(items, z, ws, out)
        if v != 0:
            return v, z
        z += 1


def check_sorted(arr, n=None) -> bool:
    """ns_scan_sorted (netsort_core.c:95-100) on the device."""
    import torch
    items, _ = _items_on_device(arr, n)
    nn = items.shape[0]
    if nn < 2:
        return True
    out = torch.empty(1, dtype=torch.int32, device=items.device)
    with torch.cuda.device(items.device):
        check(lib().nsg_scan_sorted(items.data_ptr(), 8, 16, nn, out.data_ptr(),
                                    current_stream_handle(items.device)))
    return int(out.item()) == 0


def hybrid_stats(spec, arr):
    raise ConfigurationError("hybrid quicksort is a single-array CPU sorter: out of scope of the device lane")


def measure_one_array_repeat(spec, size, iterations, seed):
    raise ConfigurationError("OneArrayRepeat times one array per call on a CPU core: use measure_array_in_row "
                             "(batched) on the device lane")


def measure_array_in_row(spec, size, narrays, seed) -> int:
    """ns_measure_air (netsort_core.c:606-659) on the device: fill
    narrays*size items from the LCG (nsg_fill_lcg), sort a throwaway copy of
    the first subarray (warm-up), then time ONE batched sort of all narrays
    contiguous subarrays with CUDA events; returns nanoseconds (TIMER_KIND).

    Verification replaces the std::sort reference copy: every subarray must be
    non-decreasing by key and a permutation of its input (key, ref) pairs
    (nsg_verify_rows, REF order) -- stronger than the reference's key equality
    + per-array ref sum/xor.  Status mapping as the reference: a network with
    size outside 2..16 (size >= 2) -> UnsupportedSize; a failed check ->
    CorrectnessFailure(seed)."""
    import torch
    size, narrays = int(size), int(narrays)
    if size < 1 or narrays < 1:
        raise ConfigurationError("size and narrays must be >= 1")
    if spec[0] == registry.KIND_NETWORK and size >= 2 and not 2 <= size <= 16:
        raise UnsupportedSize("network sorters cover 2..16 items")
    l = lib()
    dev = torch.device("cuda")
    big = torch.empty((narrays, size, 2), dtype=torch.int64, device=dev)
    fill_items(big, seed)
    inp = big.clone()
    warm = big[:1].clone()
    run_sorter_many(spec, warm)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    run_sorter_many(spec, big)
    ev1.record()
    ev1.synchronize()
    ns = int(round(ev0.elapsed_time(ev1) * 1e6))
    ki, pi = inp[..., 0].contiguous(), inp[..., 1].contiguous()
    ko, po = big[..., 0].contiguous(), big[..., 1].contiguous()
    order = registry.DeviceOrder(key_dtype=registry.KEY_U64, payload_dtype=registry.PAY_U64,
                                 descending=0, tie_mode=registry.TIE_REF)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    check(l.nsg_verify_rows(make_spec(spec, order), ki.data_ptr(), pi.data_ptr(), ko.data_ptr(), po.data_ptr(),
                            narrays, size, bad.data_ptr(), current_stream_handle(dev)))
    if int(bad.item()) != 0:
        from .errors import CorrectnessFailure
        raise CorrectnessFailure("sorted-check or fingerprint mismatch", seed=seed)
    return ns
